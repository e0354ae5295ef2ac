# does compute-sanitizer instrument libfo's kernels? wall time of the driver
# plain vs under racecheck / memcheck with the kernel filter (dev tool)
python -m paper_2204_04321_b200._build > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
t() { local s=$(date +%s.%N); "$@" > /tmp/out.txt 2>&1; local e=$(date +%s.%N); echo "$(python -c "print(round($e - $s, 1))") s: $* | $(grep -E 'SUMMARY|done' /tmp/out.txt | tr '\n' ' ')"; }
t python tools/sanitize_driver.py C2
t $CS --tool racecheck --kernel-name kns=N2fo python tools/sanitize_driver.py C2
t $CS --tool racecheck --kernel-name kns=ka_ws_kernel python tools/sanitize_driver.py C2
t $CS --tool memcheck --kernel-name kns=ka_ws_kernel python tools/sanitize_driver.py C2
t $CS --tool racecheck python tools/sanitize_driver.py C2
