timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "run_host" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python tools/summ.py new < gpurun_out/bench.json
