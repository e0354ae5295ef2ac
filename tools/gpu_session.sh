# scratch GPU session script (the command of the current gpurun call)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tmem tools/microbench_tmem.cu && /tmp/mb_tmem | tee gpurun_out/microbench_tmem.txt
python -m paper_2204_04321_b200._build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in C1 C2; do
  for tool in racecheck initcheck; do
    extra=""; [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 1500 $CS --tool $tool $extra --kernel-name kns=N2fo --print-limit 50 python tools/sanitize_driver.py $cfg > gpurun_out/sanitize_${tool}_${cfg}.txt 2>&1
    echo "$tool $cfg rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_driver .* done' gpurun_out/sanitize_${tool}_${cfg}.txt | tr '\n' ' ')"
  done
done
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee gpurun_out/pytest_gpu_r02a.txt
