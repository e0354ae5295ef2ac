# split-element experiment: parity subset + timing vs the one-thread element (dev tool)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -m paper_2204_04321_b200._build --force > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "workloads or layer_counts or single_triangle or high_degree or partitioned_assembly or symmetry or c3_full or bitwise" 2>&1 | tail -15
bash tools/gpu_variants.sh "" "-DFO_SPLIT_ELEMENT=0" "-DFO_UNROLL_SA=2 -DFO_UNROLL_SB=2"
