# A/B timing of compile-time variants on the tetrahedral path (C3, three tets
# per prism), alternating builds, with the tetrahedral parity tests per variant
# (dev tool).  usage: bash tools/gpu_ab_tet.sh ROUNDS "FLAGS_A" "FLAGS_B" ...
N=${1:-2}; shift
for v in "$@"; do
  FO_EXTRA_NVCC_FLAGS="$v" python -m paper_2204_04321_b200._build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "[$v] tests: $(FO_EXTRA_NVCC_FLAGS="$v" timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tet" 2>&1 | tail -1)"
done
for r in $(seq 1 $N); do
  for v in "$@"; do
    FO_EXTRA_NVCC_FLAGS="$v" python -m paper_2204_04321_b200._build > /dev/null 2>&1 || continue
    echo "[$v] $(FO_EXTRA_NVCC_FLAGS="$v" timeout 300 python tools/tet_quick.py 2>&1 | grep 'scatter 0')"
  done
done
