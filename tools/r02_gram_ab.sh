# K3 A/B on one box: the column-slot form (default), the tile form for every M (lib_gv1) and
# the column-slot form for every M (lib_g2all); N sweep at M = 8; per-unit timeline (lib_gprof).
# Variants: python tools/build_variant.py gv1 -DFASTRON_G2_MAXMP=0; g2all -DFASTRON_G2_MAXMP=32;
# gprof -DFASTRON_GRAM_PROF=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_train.py tests/test_gpu_joint.py tests/test_gpu_lazy.py -q -x -rf > gpurun_out/gram_ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gram_ab_tests.log
tail -3 gpurun_out/gram_ab_tests.log
for r in 1 2; do FASTRON_LIB=build/variants/lib_g2all.so python tools/gram_time.py >> gpurun_out/gram_ab.log 2>&1;
  python tools/gram_time.py >> gpurun_out/gram_ab.log 2>&1
  FASTRON_LIB=build/variants/lib_gv1.so python tools/gram_time.py >> gpurun_out/gram_ab.log 2>&1
done
NS=2560,5000,10240,20000 python tools/gram_sweep.py >> gpurun_out/gram_ab.log 2>&1
FASTRON_LIB=build/variants/lib_gprof.so NS=5000 python tools/gram_sweep.py > gpurun_out/gprof_raw.log 2>&1
python tools/gram_prof_an.py gpurun_out/gprof_raw.log >> gpurun_out/gram_ab.log; rm gpurun_out/gprof_raw.log
cat gpurun_out/gram_ab.log
