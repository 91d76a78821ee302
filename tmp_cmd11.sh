timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_e.json 2>gpurun_out/bench_e.err; echo rc=$?
