python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python tools/stack_indep.py 4096 4096 3 0.0045 64
python tools/stack_indep.py 11008 4096 3 0.0045 32
python tools/stack_indep.py 4096 11008 3 0.0045 32
python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
