nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes2 tools/micro/pipes2.cu && /tmp/pipes2 > gpurun_out/pipes2b.txt 2>&1
for s in "--d 128 --bits 3" "--d 128 --bits 4" "--d 512 --bits 3" "--d 128 --bits 2"; do
  echo "== $s sustained"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels rt q rte --only base fhadd fhaddb3fma b3fma opsreg12 base
  echo "== $s burst"; python tools/variants.py time $s --dtype f16 --variant full --kernels rt q rte --only base fhadd fhaddb3fma b3fma opsreg12 base
done > gpurun_out/var1.txt 2>&1
cat gpurun_out/var1.txt
