# A/B timing of compile-time variants on C3 R + J, alternating builds to
# average out box-to-box and run-to-run noise (dev tool)
# usage: bash tools/gpu_ab.sh ROUNDS "FLAGS_A" "FLAGS_B" ...
N=${1:-3}; shift
for r in $(seq 1 $N); do
  for v in "$@"; do
    FO_EXTRA_NVCC_FLAGS="$v" python -m paper_2204_04321_b200._build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
    echo "[$v] $(FO_EXTRA_NVCC_FLAGS="$v" FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1)"
  done
done
