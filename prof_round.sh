#!/bin/bash
# One GPU profiling round: tests, bench (ours + reference arm), launch list, ncu --set full
# of the top kernels.  Usage: bash prof_round.sh <tag>   (outputs in gpurun_out/<tag>/)
T=${1:-r1}
O=gpurun_out/$T
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-others --no-cpu > $O/b_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-others --no-cpu > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/prof_cases.py harvest --reps 1 --N 4194304 > $O/h_plain.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:harvest_poly -s 1 -c 1 -o $O/harvest \
  python tools/prof_cases.py harvest --reps 1 --N 4194304 > $O/ncu_h.log 2>&1; echo "ncu harvest rc=$?"
timeout 300 python tools/prof_cases.py c5step --reps 50 --fma > $O/c5s_plain.json 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lin_pernode_t -s 2 -c 1 -o $O/c5step \
  python tools/prof_cases.py c5step --reps 50 --fma > $O/ncu_c5s.log 2>&1; echo "ncu c5step rc=$?"
ls $O
