python - <<'PY' > gpurun_out/qjl_time.log 2>&1
import torch, iqsynth, paper_2603_28430_b200 as iq
for d in (128, 256, 512):
    for bits in (2, 3, 4):
        n = 1 << 20
        p = iq.iq_make_params_qjl(d, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
        x = iqsynth.device_unit_vectors(n, d, 7, torch.float16, "cuda")
        codes, norms, qj, rn = iq.iq_quantize_qjl(p, x)
        for i in range(3): iq.iq_quantize_qjl(p, x, codes, norms, qj, rn)
        torch.cuda.synchronize()
        def tm(fn):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(10): fn()
            e1.record(); torch.cuda.synchronize()
            return e0.elapsed_time(e1) / 10 * 1e3
        us = tm(lambda: iq.iq_quantize_qjl(p, x, codes, norms, qj, rn))
        uq = tm(lambda: iq.iq_quantize(p, x, codes, norms))
        b = n * (d * 2 + d * bits // 8 + 4 + d // 8 + 4)
        print(f"qjl d={d} b={bits}: {us:.1f} us (quantize alone {uq:.1f})  {b/us/1e3:.0f} GB/s  frac {b/us/1e3/6545:.3f}  tensor {n*4*d*d/us/1e6:.0f} TFLOP/s", flush=True)
PY
cat gpurun_out/qjl_time.log
python tools/variants.py time --d 128 --bits 3 --dtype f16 --variant full --kernels qjl --only base qjltc base qjltc
