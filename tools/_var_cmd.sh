for s in "--d 128 --bits 3" "--d 128 --bits 4" "--d 512 --bits 4" "--d 256 --bits 3"; do
  echo "== $s"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels rt q rte --only base b3fma stage64 pu2 b3fma64 b3fmapu2 grid3 opsreg nwc12 nwc20 base
done
