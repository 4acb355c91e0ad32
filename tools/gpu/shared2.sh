export IQ_BENCH_SHARED_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --preset cfg3 --steps 10 --warmup 3 --no-sweep --no-cpu --no-kernels --no-traffic > gpurun_out/shared2_cfg3.json 2> gpurun_out/shared2_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --no-sweep --no-cpu --no-kernels --no-traffic > gpurun_out/shared2_weak.json 2> gpurun_out/shared2_weak.err; echo "weak rc=$?"
tail -2 gpurun_out/shared2_cfg3.err; tail -c 1500 gpurun_out/shared2_cfg3.json; echo; tail -c 800 gpurun_out/shared2_weak.json
