# hexahedral path: parity + timing of compile-time variants (dev tool)
python -m paper_2204_04321_b200._build --force > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_newton.py -m gpu -x -q -k "hex" 2>&1 | tail -2
for F in "$@"; do
  FO_EXTRA_NVCC_FLAGS="$F" python -m paper_2204_04321_b200._build --force > /dev/null 2>&1
  echo "[$F] $(timeout 300 python tools/hex_quick.py | tr '\n' ' ')"
done
