timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py tests/test_gpu_append.py tests/test_gpu_sets.py -x -q > gpurun_out/grid2.log 2>&1; echo "rc=$?" >> gpurun_out/grid2.log; tail -2 gpurun_out/grid2.log
for s in "--d 128 --bits 4" "--d 512 --bits 4"; do
  echo "== $s sustained"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels rt q rte --only base gridscalar base gridscalar
  echo "== $s burst"; python tools/variants.py time $s --dtype f16 --variant full --kernels rt q rte --only base gridscalar base gridscalar
done
