python -m pytest tests -m gpu -x -q > gpurun_out/gputest6.log 2>&1; echo rc=$? >> gpurun_out/gputest6.log
tail -2 gpurun_out/gputest6.log
for s in "--d 128 --bits 2" "--d 256 --bits 2" "--d 512 --bits 2" "--d 128 --bits 1"; do
  echo "== $s"; python tools/variants.py time $s --dtype f16 --variant full --sustained 0.5 --kernels rt rte --only base stage16 base stage16
done
python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench rc=$?
