set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r02a.log
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"; cat gpurun_out/bench_r02a.json | head -c 600
timeout 600 bash tools/launches.sh r02a > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 bash tools/prof_fields.sh r02a k_rows_pc_tma k_cols; 
timeout 900 bash tools/prof_feat.sh k_desc_main k_fast_nms
timeout 600 bash tools/prof_gemm.sh
ls gpurun_out
