timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/par.log 2>&1; echo "rc=$?" >> gpurun_out/par.log; tail -3 gpurun_out/par.log
