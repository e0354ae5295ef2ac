# usage: bash tools/gpu_prof.sh <tag> [extra nvcc flags]
# profile the R + J path on C3: launch list (per-kernel times) and one
# ncu --set full capture of ka_ws_kernel
FO_EXTRA_NVCC_FLAGS="$2" python -m paper_2204_04321_b200._build --force 2>&1 | tail -1
mkdir -p gpurun_out
export FO_EXTRA_NVCC_FLAGS="$2"
FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tee gpurun_out/quick_$1.txt
FO_SCATTERS=0 FO_WHAT=jacobian timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python tools/quick_time.py C3 > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/launches_$1.csv | head -8
FO_SCATTERS=0 FO_WHAT=jacobian timeout 900 ncu --set full --clock-control none --import-source on -k regex:ka_ws_kernel -s 2 -c 1 -o gpurun_out/prof_$1 python tools/quick_time.py C3 > gpurun_out/ncu_$1.txt 2>&1
tail -2 gpurun_out/ncu_$1.txt
