for cfg in "32 256" "32 384" "64 512" "64 768" "128 1024"; do set -- $cfg
python tools/prof_cases.py c4 --reps 10 --tile $2 --k 1 --threads $1
python tools/prof_cases.py c4 --reps 10 --tile $2 --k 1 --threads $1 --fma
python tools/prof_cases.py c3 --reps 20 --tile $2 --k 1 --threads $1
done
for cfg in "32 256 8" "32 256 16" "64 512 16" "32 512 32"; do set -- $cfg
python tools/prof_cases.py c2 --reps 500 --tile $2 --k $3 --threads $1 --fma
done
python tools/prof_cases.py c1 --reps 2000
