python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_full.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_full.log
tail -3 gpurun_out/gputest_full.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-e2e --no-kernels --no-traffic > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o gpurun_out/r02_rt python tools/launch_kernels.py --kernel roundtrip --reps 2 > gpurun_out/ncu_rt_final.log 2>&1
