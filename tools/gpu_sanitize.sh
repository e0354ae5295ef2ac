# compute-sanitizer over every libfo kernel (tools/sanitize_driver.py) on C1 and C2:
# memcheck, racecheck, synccheck, initcheck; logs -> gpurun_out/sanitize_<tool>_<cfg>.txt
# usage (on the GPU box): bash tools/gpu_sanitize.sh
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
python -m paper_2204_04321_b200._build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for cfg in C1 C2; do
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 1500 $CS --tool $tool $extra --kernel-name kns=N2fo \
      --print-limit 50 python tools/sanitize_driver.py $cfg > gpurun_out/sanitize_${tool}_${cfg}.txt 2>&1
    echo "$tool $cfg rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_driver' gpurun_out/sanitize_${tool}_${cfg}.txt | tr '\n' ' ')"
  done
done
