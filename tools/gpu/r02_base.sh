set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 2 -o gpurun_out/base_rt python tools/launch_kernels.py --kernel roundtrip --reps 2 > gpurun_out/ncu_rt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 2 -o gpurun_out/base_q python tools/launch_kernels.py --kernel quantize --reps 2 > gpurun_out/ncu_q.log 2>&1
ls -la gpurun_out
