mkdir -p gpurun_out/r1e
python bench.py --steps 5 --warmup 3 > gpurun_out/r1e/bench.json 2> gpurun_out/r1e/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1e/bench_ref.json 2> gpurun_out/r1e/bench_ref.err; echo ref rc=$?
python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1e/b_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1e/launches.csv python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1e/ncu_launch.log 2>&1
python tools/prof_cases.py harvest --reps 1 --N 1048576 && ncu --set full --clock-control none --import-source on -k regex:harvest_quad -s 1 -c 1 -o gpurun_out/r1e/harvest python tools/prof_cases.py harvest --reps 1 --N 1048576 > gpurun_out/r1e/ncu_h.log 2>&1
python tools/prof_cases.py c5step --reps 32 && ncu --set full --clock-control none --import-source on -k regex:lin_pernode_tb -s 2 -c 1 -o gpurun_out/r1e/c5step python tools/prof_cases.py c5step --reps 32 > gpurun_out/r1e/ncu_c5s.log 2>&1
python tools/prof_cases.py c4 --reps 2 --N 4194304 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r1e/c4 python tools/prof_cases.py c4 --reps 2 --N 4194304 > gpurun_out/r1e/ncu_c4.log 2>&1
python tools/prof_cases.py c3 --reps 2 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r1e/c3 python tools/prof_cases.py c3 --reps 2 > gpurun_out/r1e/ncu_c3.log 2>&1
ls gpurun_out/r1e
