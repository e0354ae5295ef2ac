# one build -> measure iteration on the GPU box (dev tool): build, the GPU
# parity + halo tests, then C3 timings of the R + J path for each variant
# given as extra nvcc flags (";"-separated; "" = the default build)
# usage: bash tools/gpu_iter.sh TAG "VARIANT1;VARIANT2"
set -x
TAG=${1:-it}
mkdir -p gpurun_out
python -m paper_2204_04321_b200._build > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 420 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -x -q 2>&1 | tail -5 | tee gpurun_out/tests_$TAG.txt
FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -2 | tee gpurun_out/time_$TAG.txt
IFS=';' read -ra VS <<< "${2:-}"
for v in "${VS[@]}"; do
  [ -z "$v" ] && continue
  FO_EXTRA_NVCC_FLAGS="$v" python -m paper_2204_04321_b200._build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "variant: $v" | tee -a gpurun_out/time_$TAG.txt
  FO_EXTRA_NVCC_FLAGS="$v" FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1 | tee -a gpurun_out/time_$TAG.txt
done
