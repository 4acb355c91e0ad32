timeout 900 python -m pytest tests/test_gpu_qjl.py tests/test_gpu_attn.py tests/test_gpu_bf16.py -x -q > gpurun_out/qjl4.log 2>&1; echo "rc=$?" >> gpurun_out/qjl4.log
tail -2 gpurun_out/qjl4.log
for s in "--d 128 --bits 3" "--d 128 --bits 2" "--d 64 --bits 3"; do
python tools/variants.py time $s --dtype f16 --variant full --kernels qjl --only base qjlhint base qjlhint
done
