python -m pytest tests -m gpu -x -q > gpurun_out/gputest5.log 2>&1; echo rc=$? >> gpurun_out/gputest5.log
tail -2 gpurun_out/gputest5.log
python tools/attn_bench.py --d 64 --bits 3 --variant full --heads 256 2>&1 | tail -1
python tools/attn_bench.py --d 128 --bits 3 --variant full --heads 256 2>&1 | tail -1
python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench rc=$?
