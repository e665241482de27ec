# ncu --set full of the column-slot K3 at cfg3 (with source) and of the tile form at cfg5
mkdir -p gpurun_out
NS=5000 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gram2 -s 2 -c 1 -o gpurun_out/gram2_cfg3 -f python tools/gram_sweep.py > gpurun_out/gram_ncu.log 2>&1
tail -2 gpurun_out/gram_ncu.log
