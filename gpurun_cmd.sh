python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for m in multiply quad; do for s in 1 4; do python tools/prof_cases.py harvest --method $m --N 4194304 --s $s --reps 5; done; done
