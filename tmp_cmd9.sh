mkdir -p gpurun_out/r1c
python tools/prof_cases.py harvest --reps 1 --N 1048576 && ncu --set full --clock-control none --import-source on -k regex:harvest_quad -s 1 -c 1 -o gpurun_out/r1c/harvest_quad python tools/prof_cases.py harvest --reps 1 --N 1048576 > gpurun_out/r1c/ncu_h.log 2>&1
python tools/prof_cases.py c5step --reps 3 && ncu --set full --clock-control none --import-source on -k regex:lin_pernode -s 3 -c 1 -o gpurun_out/r1c/c5step python tools/prof_cases.py c5step --reps 3 > gpurun_out/r1c/ncu_c5s.log 2>&1
ls gpurun_out/r1c
