python -m paper_2204_04321_b200._build > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kh_patch_kernel -s 3 -c 1 -o gpurun_out/prof_hex1 python tools/hex_quick.py > gpurun_out/ncu_hex1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_hex1.csv python tools/hex_quick.py > /dev/null 2>&1
tail -2 gpurun_out/ncu_hex1.txt
