for s in "--d 128 --bits 3" "--d 128 --bits 4" "--d 512 --bits 4" "--d 128 --bits 2"; do
  echo "== $s"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels dq q rt --only base
done
