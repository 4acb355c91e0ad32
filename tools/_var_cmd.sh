python -m pytest tests -m gpu -x -q > gpurun_out/gputest3.log 2>&1; echo rc=$? >> gpurun_out/gputest3.log
for s in "--d 128 --bits 3" "--d 128 --bits 2" "--d 512 --bits 3"; do
  echo "== $s"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels q rte --only base wordcodes base wordcodes
done
python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench rc=$?
