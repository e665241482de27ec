# K5 A/B (run under gpurun from the repo root): LIBS builds on cfg3, N = 1000 and 8446
mkdir -p gpurun_out
L=gpurun_out/train_ab.log; : > $L
for lib in $LIBS; do
  echo "== lib: $lib" >> $L
  FASTRON_LIB=$lib timeout 300 python tools/train_sweep.py 5 8 >> $L 2>&1
  FASTRON_LIB=$lib TRAIN_N=1000 timeout 300 python tools/train_sweep.py 1 >> $L 2>&1
  FASTRON_LIB=$lib TRAIN_N=8446 timeout 300 python tools/train_sweep.py 9 >> $L 2>&1
  FASTRON_LIB=$lib TRAIN_N=20000 timeout 300 python tools/train_sweep.py 16 >> $L 2>&1
done
cut -c1-75 $L
