timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 300 python tools/chain_nodep.py 2>&1 | tail -2
echo "$(timeout 120 python tools/stack_indep.py 4096 4096 3 0.05 32 2>&1 | tail -1)"
echo "$(timeout 120 python tools/stack_indep.py 11008 4096 3 0.0045 32 2>&1 | tail -1)"
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python tools/summ.py now
