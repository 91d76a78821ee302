timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/prof_cases.py harvest --reps 2 --N 1048576
for th in 128 256; do for t in 256 512 1024; do python tools/prof_cases.py c4 --reps 10 --tile $t --k 1 --threads $th; python tools/prof_cases.py c3 --reps 20 --tile $t --k 1 --threads $th; done; done
python tools/prof_cases.py c4 --reps 10 --tile 512 --k 1 --threads 128 --fma
python tools/prof_cases.py c3 --reps 20 --tile 512 --k 1 --threads 128 --fma
for k in 4 8 16; do python tools/prof_cases.py c2 --reps 500 --k $k --tile 512; python tools/prof_cases.py c2 --reps 500 --k $k --tile 256 --threads 128; done
