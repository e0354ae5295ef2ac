# full round check on one B200: build, gpu tests, smoke, one ncu --set full
# capture of the top kernel (-> profiles/ncu_summary.json on the box, read by
# bench.py; gpurun merges only gpurun_out/ back, so copy
# gpurun_out/ncu_summary.json to profiles/ here and commit it),
# the ncu launch list of the bench command, then the bench (ours + reference)
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke_$TAG.txt
timeout 900 ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none --import-source on -k regex:ka_ws_kernel -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$TAG.txt 2>&1
tail -2 gpurun_out/ncu_$TAG.txt
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep C3 4797110 gpurun_out/ncu_summary.json && cp gpurun_out/ncu_summary.json profiles/ncu_summary.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_$TAG.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 2>&1 | tail -2 | tee gpurun_out/bench_ref_$TAG.txt
