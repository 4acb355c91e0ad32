# Round-2 (third session) evidence, part B: compute-sanitizer on the kernels
# changed this session (register operators, byte-piece code stores).
OUT=gpurun_out/r02_sanitize4; mkdir -p $OUT
CS="compute-sanitizer --error-exitcode 17 --print-limit 50 --target-processes all"
timeout 1500 $CS --tool memcheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py::test_parity_grid tests/test_gpu_parity.py::test_ragged_n tests/test_gpu_append.py > $OUT/memcheck_stage1.log 2>&1; echo "memcheck(stage1, append) rc=$?" >> $OUT/summary.txt
timeout 1500 $CS --tool memcheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_qjl.py -k "128" > $OUT/memcheck_qjl.log 2>&1; echo "memcheck(qjl d<=128) rc=$?" >> $OUT/summary.txt
timeout 2400 $CS --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py -k "test_parity_grid and (64 or 512) and (3- or 4-)" > $OUT/racecheck_stage1.log 2>&1; echo "racecheck(stage1) rc=$?" >> $OUT/summary.txt
timeout 900 $CS --tool synccheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py -k "test_parity_grid and 128 and 3-" > $OUT/synccheck_stage1.log 2>&1; echo "synccheck(stage1) rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt
for f in $OUT/*.log; do echo "== $f"; tail -3 $f; done
