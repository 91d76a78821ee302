timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c4 c3; do python tools/prof_cases.py $c --reps 10; python tools/prof_cases.py $c --reps 10 --fma; done
for cfg in "224 1024" "256 1200" "160 768" "96 448"; do set -- $cfg; python tools/prof_cases.py c4 --reps 10 --tile $2 --k 1 --threads $1; python tools/prof_cases.py c3 --reps 10 --tile $2 --k 1 --threads $1; done
python tools/prof_cases.py c2 --reps 500
python tools/prof_cases.py c2 --reps 500 --fma
