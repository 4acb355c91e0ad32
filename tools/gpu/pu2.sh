for s in "--d 128 --bits 3" "--d 128 --bits 4" "--d 512 --bits 3"; do
  echo "== $s burst"; python tools/variants.py time $s --dtype f16 --variant full --kernels rt q rte --only base pu2 pu2w8 pu2w12 base
done
echo "== d128 b3 sustained"; python tools/variants.py time --d 128 --bits 3 --dtype f16 --variant full --sustained 0.5 --kernels rt q --only base pu2w8 pu2w12 base
