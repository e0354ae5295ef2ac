# one ncu --set full capture of the R + J assembly kernel (ka_ws_kernel) at C3
# plus the compute-sanitizer suite (tools/gpu_sanitize.sh); usage: bash tools/gpu_prof_sanitize.sh TAG
set -x
TAG=${1:-r02}
mkdir -p gpurun_out
python -m paper_2204_04321_b200._build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none --import-source on -k regex:ka_ws_kernel -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$TAG.txt 2>&1
tail -2 gpurun_out/ncu_$TAG.txt
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep C3 4797110 gpurun_out/ncu_summary_$TAG.json > /dev/null
bash tools/gpu_sanitize.sh
