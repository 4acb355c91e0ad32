python -m pytest tests -m gpu -x -q > gpurun_out/gputest4.log 2>&1; echo rc=$? >> gpurun_out/gputest4.log
python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench rc=$?
