mkdir -p gpurun_out/r1d
python bench.py --steps 5 --warmup 3 > gpurun_out/r1d/bench.json 2> gpurun_out/r1d/bench.err; echo bench rc=$?
python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1d/b_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d/launches.csv python bench.py --steps 1 --warmup 1 --no-others --no-cpu > gpurun_out/r1d/ncu_launch.log 2>&1
ls gpurun_out/r1d
