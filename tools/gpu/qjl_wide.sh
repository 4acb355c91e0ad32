timeout 900 python -m pytest tests/test_gpu_qjl.py -x -q > gpurun_out/qjl_wide.log 2>&1; echo "rc=$?" >> gpurun_out/qjl_wide.log
tail -30 gpurun_out/qjl_wide.log
python - <<'PY' >> gpurun_out/qjl_wide.log 2>&1
import torch, iqsynth, paper_2603_28430_b200 as iq
for d in (128, 256, 512):
    for bits in (2, 3, 4):
        n = 1 << 20
        p = iq.iq_make_params_qjl(d, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
        x = iqsynth.device_unit_vectors(n, d, 7, torch.float16, "cuda")
        codes, norms, qj, rn = iq.iq_quantize_qjl(p, x)
        for i in range(3): iq.iq_quantize_qjl(p, x, codes, norms, qj, rn)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10): iq.iq_quantize_qjl(p, x, codes, norms, qj, rn)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        b = n * (d * 2 + d * bits // 8 + 4 + d // 8 + 4)
        print(f"qjl d={d} b={bits}: {us:.1f} us  {b/us/1e3:.0f} GB/s  frac {b/us/1e3/6545:.3f}  tensor {n*4*d*d/us/1e6:.0f} TFLOP/s")
PY
tail -12 gpurun_out/qjl_wide.log
