# per compile-time variant: C3 R + J time, hexahedra time, and the DRAM / L2
# counters of ka_ws_kernel (dev tool).  usage: bash tools/gpu_variants_dram.sh TAG "FLAGS_A" "FLAGS_B" ...
TAG=$1; shift
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sector_hit_rate.pct
for v in "$@"; do
  FO_EXTRA_NVCC_FLAGS="$v" python -m paper_2204_04321_b200._build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "[$v] $(FO_EXTRA_NVCC_FLAGS="$v" FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1)"
  echo "[$v] $(FO_EXTRA_NVCC_FLAGS="$v" timeout 300 python tools/hex_quick.py 2>&1 | grep 'owner hex RJ')"
  FO_EXTRA_NVCC_FLAGS="$v" FO_SCATTERS=0 FO_WHAT=jacobian timeout 600 ncu --metrics $M --clock-control none -k regex:ka_ws_kernel -s 3 -c 1 python tools/quick_time.py C3 2>&1 | grep -E "dram__|lts__|gpu__" | sed "s/^/[$v] /"
done 2>&1 | tee gpurun_out/variants_$TAG.txt
