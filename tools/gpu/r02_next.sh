python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_qjl.py tests/test_gpu_append.py -x -q > gpurun_out/next_tests.log 2>&1; echo "rc=$?" >> gpurun_out/next_tests.log
for args in "--d 128 --bits 3 --variant full" "--d 128 --bits 4 --variant fast" "--d 256 --bits 3 --variant full" "--d 64 --bits 3 --variant full"; do
  python tools/attn_bench.py $args >> gpurun_out/attn_r02.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qjl_sketch -c 1 -o gpurun_out/sketch256b python tools/launch_kernels.py --kernel quantize_qjl --d 256 --reps 1 > gpurun_out/ncu_sketch2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn -c 1 -o gpurun_out/attn_b python tools/launch_kernels.py --kernel attention --reps 1 > gpurun_out/ncu_attn2.log 2>&1
tail -2 gpurun_out/smoke2.log; tail -2 gpurun_out/next_tests.log; cat gpurun_out/attn_r02.jsonl
compute-sanitizer --error-exitcode 17 --print-limit 20 --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_qjl.py -k "ragged and 512" > gpurun_out/racecheck_sketch512.log 2>&1; echo "racecheck(sketch 512) rc=$?" >> gpurun_out/racecheck_sketch512.log
tail -3 gpurun_out/racecheck_sketch512.log
