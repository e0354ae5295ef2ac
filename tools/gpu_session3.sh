python -m paper_2204_04321_b200._build --force 2>&1 | tail -1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
timeout 600 python tools/quick_time.py C3 2>&1 | tee gpurun_out/quick_c3.txt
FO_SCATTERS=0 FO_WHAT=jacobian timeout 600 ncu --set full --clock-control none --import-source on -k regex:ka_patch_kernel -s 1 -c 1 -o gpurun_out/prof_patchJ python tools/quick_time.py C3 > gpurun_out/ncu_log.txt 2>&1
FO_SCATTERS=0 FO_WHAT=residual timeout 600 ncu --set full --clock-control none --import-source on -k regex:ka_patch_kernel -s 1 -c 1 -o gpurun_out/prof_patchR python tools/quick_time.py C3 >> gpurun_out/ncu_log.txt 2>&1
tail -3 gpurun_out/ncu_log.txt
