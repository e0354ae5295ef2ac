# claims vs zero fill: GPU tests in the default build, then A/B timings of the
# wedge (C3) and hexahedral paths against -DFO_NO_CLAIM, and DRAM / RED counters
set -x
mkdir -p gpurun_out
python -m paper_2204_04321_b200._build > gpurun_out/build_claim.log 2>&1 || { tail -30 gpurun_out/build_claim.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/tests_claim.txt
bash tools/gpu_ab.sh 2 "" "-DFO_NO_CLAIM" 2>&1 | tee gpurun_out/ab_claim.txt
bash tools/gpu_ab_hex.sh 1 "" "-DFO_NO_CLAIM" 2>&1 | tee -a gpurun_out/ab_claim.txt
python -m paper_2204_04321_b200._build > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_write.sum
FO_SCATTERS=0 FO_WHAT=jacobian timeout 600 ncu --metrics $M --clock-control none -k regex:ka_ws_kernel -s 3 -c 1 python tools/quick_time.py C3 2>&1 | grep -E "ka_ws|gpu__|dram__|lts__" | tee gpurun_out/ncu_claim.txt
timeout 600 ncu --metrics $M --clock-control none -k regex:kh_patch_kernel -s 3 -c 1 python tools/hex_quick.py 2>&1 | grep -E "kh_patch|gpu__|dram__|lts__" | tee -a gpurun_out/ncu_claim.txt
