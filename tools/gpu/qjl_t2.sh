timeout 600 python -m pytest tests/test_gpu_qjl.py -x -q -k "wide or ragged" > gpurun_out/qjl_t2.log 2>&1; echo "rc=$?" >> gpurun_out/qjl_t2.log; tail -2 gpurun_out/qjl_t2.log
bash tools/gpu/qjl_time.sh 2>&1 | head -9
