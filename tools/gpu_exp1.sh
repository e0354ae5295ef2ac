# experiment: element-only time (phase B compiled out; results not valid)
FO_EXTRA_NVCC_FLAGS="-DFO_EXPERIMENT_NO_PHASE_B" python -m paper_2204_04321_b200._build --force 2>&1 | tail -1
FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1
python -m paper_2204_04321_b200._build --force 2>&1 | tail -1
FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1
