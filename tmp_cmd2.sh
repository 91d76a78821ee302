timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c1 c2; do python tools/prof_cases.py $c --reps 200; python tools/prof_cases.py $c --reps 200 --fma; done
for t in 512 1024 2048; do python tools/prof_cases.py c4 --reps 10 --tile $t --k 1; python tools/prof_cases.py c4 --reps 10 --tile $t --k 1 --fma; python tools/prof_cases.py c3 --reps 10 --tile $t --k 1; python tools/prof_cases.py c3 --reps 10 --tile $t --k 1 --fma; done
python tools/prof_cases.py c5step --reps 20
python tools/prof_cases.py harvest --reps 2 --N 1048576
