set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c1 c2; do python tools/prof_cases.py $c --reps 200; python tools/prof_cases.py $c --reps 200 --fma; done
for t in 256 512 1024 2048; do python tools/prof_cases.py c4 --reps 10 --tile $t --k 1; python tools/prof_cases.py c3 --reps 10 --tile $t --k 1; done
python tools/prof_cases.py c4 --reps 10 --fma; python tools/prof_cases.py c3 --reps 10 --fma
python tools/prof_cases.py c5step --reps 20
python tools/prof_cases.py harvest --reps 2 --N 1048576
python tools/prof_cases.py harvest --reps 1 --N 262144 && ncu --set full --clock-control none --import-source on -k regex:harvest_kernel -s 2 -c 1 -o gpurun_out/prof_harvest python tools/prof_cases.py harvest --reps 1 --N 262144 > gpurun_out/ncu_h.log 2>&1
python tools/prof_cases.py c4 --reps 2 --N 4194304 && ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_c4 python tools/prof_cases.py c4 --reps 2 --N 4194304 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_h.log gpurun_out/ncu_c4.log
