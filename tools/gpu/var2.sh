for s in "--d 128 --bits 3" "--d 512 --bits 4"; do
  echo "== $s sustained"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels rt --only base tpl8 tpl8w12 tpl8w20 base
  echo "== $s burst"; python tools/variants.py time $s --dtype f16 --variant full --kernels rt --only base tpl8 tpl8w12 tpl8w20 base
done > gpurun_out/var2.txt 2>&1
cat gpurun_out/var2.txt
