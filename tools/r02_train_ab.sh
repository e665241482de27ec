# K5 A/B (run under gpurun from the repo root): HEAD build vs the working tree on cfg3,
# N = 1000, 8446 and 20000, then the training GPU tests.
mkdir -p gpurun_out
L=gpurun_out/train_ab.log; : > $L
for lib in build/variants/lib_head.so build/variants/lib_v1.so paper_1910_06451_b200/libfastron_b200.so build/variants/lib_head.so build/variants/lib_v1.so paper_1910_06451_b200/libfastron_b200.so; do
  echo "== lib: $lib" >> $L
  FASTRON_LIB=$lib timeout 300 python tools/train_sweep.py 1 5 8 >> $L 2>&1
  FASTRON_LIB=$lib TRAIN_N=1000 timeout 300 python tools/train_sweep.py 1 >> $L 2>&1
  FASTRON_LIB=$lib TRAIN_N=8446 timeout 300 python tools/train_sweep.py 9 >> $L 2>&1
done
cut -c1-75 $L
