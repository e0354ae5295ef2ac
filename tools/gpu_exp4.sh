for F in "FO_EXPERIMENT_NO_GATHER -DFO_EXPERIMENT_LINEAR_STORE" "FO_EXPERIMENT_LINEAR_STORE"; do
FO_EXTRA_NVCC_FLAGS="-D$F" python -m paper_2204_04321_b200._build --force 2>&1 | tail -0
echo $F; FO_SCATTERS=0 FO_WHAT=jacobian timeout 300 python tools/quick_time.py C3 2>&1 | tail -1
done
python -m paper_2204_04321_b200._build --force 2>&1 | tail -1
