python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2500 gpurun_out/bench.json
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -c 600 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --soak 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stack_gemv -s 23 -c 1 -o gpurun_out/prof_bench python bench.py --steps 20 --warmup 3 --soak 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log
