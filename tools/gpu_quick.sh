# quick GPU check of the working tree: build, all gpu tests, C3 timing of compile-time variants (dev tool)
# usage: bash tools/gpu_quick.sh "<flags1>" "<flags2>" ...
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -m paper_2204_04321_b200._build --force > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
bash tools/gpu_variants.sh "$@"
