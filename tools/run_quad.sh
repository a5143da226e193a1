set -x
python -m pytest tests/test_gpu_stages.py tests/test_gpu_edges.py tests/test_gpu_timed.py -m gpu -q -x -k "fields or maps or median" > gpurun_out/t3.log 2>&1; echo pytest_rc=$? >> gpurun_out/t3.log
python tools/fields_timing.py --size 1024 --pairs 16 > gpurun_out/ft3.log 2>&1
python tools/fields_timing.py --size 512 --pairs 64 >> gpurun_out/ft3.log 2>&1
python tools/fields_timing.py --size 4096 --pairs 1 --iters 5 >> gpurun_out/ft3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum --clock-control none -k regex:^k_ -s 20 -c 10 --csv --log-file gpurun_out/launches_q3.csv python tools/fields_timing.py --size 1024 --pairs 16 --iters 2 > gpurun_out/ncu_q3.log 2>&1
