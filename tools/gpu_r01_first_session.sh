# round-1 first GPU session (microbench, GPU tests, first C3 timing); kept for the record (dev tool)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2204_04321_b200._build --force
mkdir -p gpurun_out
./tools/microbench_fp64 2>&1 | tee gpurun_out/microbench.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.txt
timeout 600 python tools/quick_time.py C3 2>&1 | tee gpurun_out/quick_c3.txt
