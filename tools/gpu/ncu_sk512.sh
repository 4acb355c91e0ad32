timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qjl_sketch -c 1 -o gpurun_out/sketch512 python tools/launch_kernels.py --kernel quantize_qjl --d 512 --reps 1 > gpurun_out/ncu_sk512.log 2>&1
tail -2 gpurun_out/ncu_sk512.log
