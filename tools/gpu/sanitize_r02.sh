OUT=gpurun_out/r02_sanitize2; mkdir -p $OUT
CS="compute-sanitizer --error-exitcode 17 --print-limit 50 --target-processes all"
timeout 1500 $CS --tool memcheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_qjl.py -k "wide and (3- or 4-) or ragged or special" > $OUT/memcheck_qjl_wide.log 2>&1; echo "memcheck(qjl wide) rc=$?" >> $OUT/summary.txt
timeout 900 $CS --tool synccheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_qjl.py -k "ragged or special" > $OUT/synccheck_qjl.log 2>&1; echo "synccheck(qjl) rc=$?" >> $OUT/summary.txt
timeout 1500 $CS --tool initcheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py::test_ragged_n tests/test_gpu_qjl.py tests/test_gpu_append.py -k "ragged or special or append" > $OUT/initcheck.log 2>&1; echo "initcheck rc=$?" >> $OUT/summary.txt
timeout 2400 $CS --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py -k "test_parity_grid and (64 or 512) and (3- or 4-)" > $OUT/racecheck_stage1.log 2>&1; echo "racecheck(stage1) rc=$?" >> $OUT/summary.txt
timeout 1800 $CS --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_qjl.py tests/test_gpu_attn.py -k "ragged or shapes or head_switches" > $OUT/racecheck_next.log 2>&1; echo "racecheck(next) rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt
for f in $OUT/*.log; do echo "== $f"; tail -4 $f; done
