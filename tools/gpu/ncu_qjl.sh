timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quantize_qjl -c 1 -o gpurun_out/base_qjl python tools/launch_kernels.py --kernel quantize_qjl --reps 2 > gpurun_out/ncu_qjl.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attn -c 1 -o gpurun_out/base_attn python tools/launch_kernels.py --kernel attention --reps 2 > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
