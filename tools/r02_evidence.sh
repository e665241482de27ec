# ncu evidence for K4 (edge FK + edge-mode scoring at cfg4) and the small-batch kernel; pipe peaks
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gpurun_out/pipe_peaks tools/pipe_peaks.cu && ./gpurun_out/pipe_peaks > gpurun_out/pipe_peaks.json
python tools/edge_time.py > gpurun_out/edge_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/edge_launches.csv python tools/edge_time.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"edge_fk_kernel|score_kernel" -c 4 -o gpurun_out/edge_cfg4 python tools/edge_time.py > gpurun_out/edge_ncu.log 2>&1
WL=headline NQ=1 REPS=5 ncu --set full --clock-control none --import-source on -k regex:score_small -c 1 -s 2 -o gpurun_out/small_q1_S20k python tools/cfg1_probe.py > gpurun_out/small_ncu.log 2>&1
WL=headline NQ=1 REPS=5 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python tools/cfg1_probe.py > /dev/null 2>&1
ls gpurun_out
