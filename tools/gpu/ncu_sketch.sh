timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qjl_sketch -c 1 -o gpurun_out/sketch256 python tools/launch_kernels.py --kernel quantize_qjl --d 256 --reps 1 > gpurun_out/ncu_sketch.log 2>&1
tail -3 gpurun_out/ncu_sketch.log
