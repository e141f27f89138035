timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "batched_stack or stack_chain or batched_products" 2>&1 | tail -2
for b in 1 2 4; do timeout 600 python tools/bench_stack.py --model 7b --batch $b 2>&1 | tail -1 | cut -c1-330; done
