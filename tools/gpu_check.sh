# build, all GPU tests, C3 R + J timing, hexahedral timing, and the DRAM /
# RED counters of the two patch kernels (dev tool)
# usage: bash tools/gpu_check.sh TAG
set -x
TAG=${1:-chk}
mkdir -p gpurun_out
python -m paper_2204_04321_b200._build > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee gpurun_out/tests_$TAG.txt
for i in 1 2; do FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1 | tee -a gpurun_out/time_$TAG.txt; done
timeout 300 python tools/hex_quick.py 2>&1 | grep owner | tee -a gpurun_out/time_$TAG.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_write.sum
FO_SCATTERS=0 FO_WHAT=jacobian timeout 600 ncu --metrics $M --clock-control none -k regex:ka_ws_kernel -s 3 -c 1 python tools/quick_time.py C3 2>&1 | grep -E "ka_ws|gpu__|dram__|lts__" | tee gpurun_out/ncu_$TAG.txt
timeout 600 ncu --metrics $M --clock-control none -k regex:kh_patch_kernel -s 3 -c 1 python tools/hex_quick.py 2>&1 | grep -E "kh_patch|gpu__|dram__|lts__" | tee -a gpurun_out/ncu_$TAG.txt
