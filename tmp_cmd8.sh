mkdir -p gpurun_out/r1b
python bench.py --steps 5 --warmup 3 > gpurun_out/r1b/bench.json 2> gpurun_out/r1b/bench.err; echo bench rc=$?
python tools/prof_cases.py harvest --reps 1 --N 1048576 && ncu --set full --clock-control none --import-source on -k regex:harvest_quad -s 1 -c 1 -o gpurun_out/r1b/harvest_quad python tools/prof_cases.py harvest --reps 1 --N 1048576 > gpurun_out/r1b/ncu_h.log 2>&1
python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1b/b_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b/launches.csv python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1b/ncu_launch.log 2>&1
ls gpurun_out/r1b
