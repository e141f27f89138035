timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "batched_stack or stack_chain or batched_products" 2>&1 | tail -2
timeout 600 python tools/bench_stack.py --model all --batch 2 2>&1 | cut -c1-260
timeout 600 python tools/bench_stack.py --model 7b --batch 4 2>&1 | cut -c1-260
timeout 600 python tools/bench_stack.py --model 7b 2>&1 | cut -c1-260
