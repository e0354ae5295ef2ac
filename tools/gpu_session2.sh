set -x
python -m paper_2204_04321_b200._build --force 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.txt
timeout 600 python tools/quick_time.py C3 2>&1 | tee gpurun_out/quick_c3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ka_patch_kernel -s 2 -c 1 -o gpurun_out/prof_patch python tools/quick_time.py C3 > gpurun_out/ncu_log.txt 2>&1
ls -la gpurun_out
