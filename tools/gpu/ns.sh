for s in "--d 128 --bits 3" "--d 128 --bits 4"; do
  echo "== $s burst"; python tools/variants.py time $s --dtype f16 --variant full --kernels rt q rte --only base nsplit base nsplit
done
