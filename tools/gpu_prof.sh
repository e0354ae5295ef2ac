# usage: bash tools/gpu_prof.sh <tag>   (profile the owner Jacobian kernel on C3)
python -m paper_2204_04321_b200._build --force 2>&1 | tail -1
mkdir -p gpurun_out
FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tee gpurun_out/quick_$1.txt
FO_SCATTERS=0 FO_WHAT=jacobian timeout 900 ncu --set full --clock-control none --import-source on -k regex:ka_ws_kernel -s 2 -c 1 -o gpurun_out/prof_$1 python tools/quick_time.py C3 > gpurun_out/ncu_$1.txt 2>&1
tail -2 gpurun_out/ncu_$1.txt
