# time several compile-time variants of the library on C3 (dev tool)
# usage: bash tools/gpu_variants.sh "<flags1>" "<flags2>" ...
for F in "$@"; do
  FO_EXTRA_NVCC_FLAGS="$F" python -m paper_2204_04321_b200._build --force > /dev/null 2>&1
  echo "[$F] $(FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1)"
done
python -m paper_2204_04321_b200._build --force > /dev/null 2>&1
