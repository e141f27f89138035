timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "batched" 2>&1 | tail -2
timeout 600 python tools/batch_sweep.py --shapes 4096x4096,11008x4096,4096x11008 --bits 3,4 --sparsity 0.0045 --batches 1,4,5,8,16 2>&1 | python3 -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['shape'],d['bits'],d['batch'],d['us'],d['TFLOPs'],d['speedup_vs_B_x_batch1'])
"
