timeout 900 python -m pytest tests/test_gpu_qjl.py tests/test_gpu_attn.py -x -q > gpurun_out/qjl3.log 2>&1; echo "rc=$?" >> gpurun_out/qjl3.log
tail -3 gpurun_out/qjl3.log
python tools/variants.py time --d 128 --bits 3 --dtype f16 --variant full --kernels qjl --only base qjlrn base qjlrn
python tools/variants.py time --d 64 --bits 3 --dtype f16 --variant full --kernels qjl --only base qjlrn
