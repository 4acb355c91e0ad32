python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_final.log
tail -3 gpurun_out/gputest_final.log
for i in 1 2; do timeout 900 python bench.py > gpurun_out/bench_final_$i.json 2> gpurun_out/bench_final_$i.err; echo "bench $i rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-e2e --no-kernels --no-traffic > gpurun_out/b_ncu_final.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o gpurun_out/final_rt python tools/launch_kernels.py --kernel roundtrip --reps 2 > gpurun_out/ncu_final_rt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o gpurun_out/final_q python tools/launch_kernels.py --kernel quantize --reps 2 > gpurun_out/ncu_final_q.log 2>&1
OUT=gpurun_out/final_san; mkdir -p $OUT
compute-sanitizer --error-exitcode 17 --print-limit 20 --tool racecheck --racecheck-report hazard python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py -k "test_parity_grid and (64 or 512) and (3- or 4-)" > $OUT/racecheck_stage1.log 2>&1; echo "racecheck stage1 rc=$?" >> $OUT/summary.txt
compute-sanitizer --error-exitcode 17 --print-limit 20 --tool memcheck python -m pytest -p no:cacheprovider -q -m gpu tests/test_gpu_parity.py::test_parity_grid tests/test_gpu_parity.py::test_ragged_n tests/test_gpu_append.py > $OUT/memcheck_stage1.log 2>&1; echo "memcheck stage1 rc=$?" >> $OUT/summary.txt
cat $OUT/summary.txt
