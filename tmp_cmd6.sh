python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo rc=$?; tail -3 gpurun_out/bench_r1c.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$?
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
