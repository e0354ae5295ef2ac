# scratch GPU session script (the command of the current gpurun call)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -m paper_2204_04321_b200._build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_workloads or c2_full" 2>&1 | tail -15
FO_SCATTERS=3,2 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -4
