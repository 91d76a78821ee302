python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo rc=$?
python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/b_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/prof_cases.py harvest --reps 1 --N 262144 && ncu --set full --clock-control none --import-source on -k regex:harvest_kernel -s 2 -c 1 -o gpurun_out/prof_harvest3 python tools/prof_cases.py harvest --reps 1 --N 262144 > gpurun_out/ncu_h3.log 2>&1
python tools/prof_cases.py c5step --reps 3 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_c5step python tools/prof_cases.py c5step --reps 3 > gpurun_out/ncu_c5s.log 2>&1
tail -c 400 gpurun_out/ncu_launch.log; ls -la gpurun_out
