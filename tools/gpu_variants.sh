# time several compile-time variants of the library on C3 (dev tool)
# usage: bash tools/gpu_variants.sh "<flags1>" "<flags2>" ...
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv,noheader
for F in "$@"; do
  FO_EXTRA_NVCC_FLAGS="$F" python -m paper_2204_04321_b200._build --force > /dev/null 2>&1
  nvidia-smi --query-gpu=clocks.sm --format=csv,noheader -lms 200 > /tmp/clk.txt & CP=$!
  R=$(FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1)
  kill $CP; echo "[$F] $R   sm_clk: $(sort /tmp/clk.txt | uniq -c | sort -rn | head -2 | tr '\n' ' ')"
done
python -m paper_2204_04321_b200._build --force > /dev/null 2>&1
