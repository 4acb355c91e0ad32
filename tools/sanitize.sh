#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the GPU
# parity tests (SURVEY 4.2 tier T6 on T4): every stage-1 kernel kind on the
# small grid, plus the stage-2 sketch, the decode consumer, the parameter-set
# instances and the distortion gradient.  Logs go to $OUT (default
# gpurun_out/).  Usage: tools/sanitize.sh [tool ...]
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
CS="compute-sanitizer --error-exitcode 17 --print-limit 50 --target-processes all"
# memcheck/synccheck/initcheck: the whole T4 grid and the NEXT-row kernels
GRID='tests/test_gpu_parity.py::test_parity_grid tests/test_gpu_parity.py::test_ragged_n tests/test_gpu_parity.py::test_edge_vectors'
NEXT='tests/test_gpu_qjl.py tests/test_gpu_attn.py tests/test_gpu_sets.py tests/test_gpu_learn.py tests/test_gpu_bf16.py'
# racecheck (shared-memory hazards, much slower): d in {64, 512} x bits {3, 4}
# x every variant and dtype, plus the tcgen05 kernels at small n
RACE_K='test_parity_grid and (64 or 512) and (3- or 4-)'
tools=${@:-memcheck synccheck initcheck racecheck}
for t in $tools; do
  case $t in
    racecheck)
      timeout 2400 $CS --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu \
        tests/test_gpu_parity.py -k "$RACE_K" > "$OUT/sanitize_racecheck.log" 2>&1
      echo "racecheck rc=$?" >> "$OUT/sanitize_summary.txt"
      timeout 1800 $CS --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu \
        tests/test_gpu_qjl.py tests/test_gpu_attn.py tests/test_gpu_sets.py -k "ragged or shapes or head_switches or sets_stage1" \
        > "$OUT/sanitize_racecheck_next.log" 2>&1
      echo "racecheck(next) rc=$?" >> "$OUT/sanitize_summary.txt" ;;
    *)
      timeout 2400 $CS --tool $t python -m pytest -p no:cacheprovider -q -m gpu $GRID $NEXT \
        -k "not large_batch and not kv_cache_shaped and not learning_loop" > "$OUT/sanitize_$t.log" 2>&1
      echo "$t rc=$?" >> "$OUT/sanitize_summary.txt" ;;
  esac
done
