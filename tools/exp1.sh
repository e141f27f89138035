for dbg in 0 512; do
  P=paper_2306_07629_b200/libdsq_cuda_prof.so
  echo "== $dbg"; DSQ_STACK_DBG_EXTRA=$dbg DSQ_CUDA_LIB=$P timeout 120 python tools/stack_prof.py 4096 4096 3 2>&1 | tail -2
  echo "== dbg=$dbg $(DSQ_STACK_DBG=$dbg timeout 120 python tools/stack_indep.py 4096 4096 3 2>&1 | tail -1)"
done
