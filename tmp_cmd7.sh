mkdir -p gpurun_out/r1
python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1/b_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1/launches.csv python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1/ncu_launch.log 2>&1
python tools/prof_cases.py harvest --reps 1 --N 262144 && ncu --set full --clock-control none --import-source on -k regex:harvest_kernel -s 2 -c 1 -o gpurun_out/r1/harvest python tools/prof_cases.py harvest --reps 1 --N 262144 > gpurun_out/r1/ncu_h.log 2>&1
python tools/prof_cases.py c5step --reps 3 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r1/c5step python tools/prof_cases.py c5step --reps 3 > gpurun_out/r1/ncu_c5s.log 2>&1
python tools/prof_cases.py c4 --reps 2 --N 4194304 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r1/c4 python tools/prof_cases.py c4 --reps 2 --N 4194304 > gpurun_out/r1/ncu_c4.log 2>&1
python tools/prof_cases.py c3 --reps 2 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r1/c3 python tools/prof_cases.py c3 --reps 2 > gpurun_out/r1/ncu_c3.log 2>&1
ls -la gpurun_out/r1
