"""Rate of the fused kernel over time under continuous load (power / clock
behaviour).  Launches the headline K3 back to back for --seconds and prints
the per-window kernel time (CUDA events, windows of --window launches) with
the SM clock and power sampled by NVML at the same moments.

  python tools/power_probe.py --seconds 3 --window 50
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--window", type=int, default=50)
    ap.add_argument("--idle", type=float, default=0.0, help="idle seconds before starting")
    a = ap.parse_args()
    import torch
    import pynvml
    import iqsynth
    import paper_2603_28430_b200 as iq
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    p = iq.iq_make_params(128, 3, iq.FULL, iqsynth.PARAMS_SEED, device=0)
    xs = [iqsynth.device_unit_vectors(1 << 20, 128, 7 + j, torch.float16, "cuda") for j in range(2)]
    ys = [torch.empty_like(x) for x in xs]
    s = torch.cuda.current_stream()
    for i in range(5):
        iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], stream=s)
    torch.cuda.synchronize()
    time.sleep(a.idle)
    t0 = time.time()
    k = 0
    while time.time() - t0 < a.seconds:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(a.window):
            iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1], stream=s)
        e1.record(s)
        e1.synchronize()
        us = e0.elapsed_time(e1) / a.window * 1e3
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mclk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
        reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        print(f"t={time.time() - t0:6.3f}s  {us:7.1f} us/launch  sm={clk} MHz mem={mclk} MHz  "
              f"power={pw:6.1f} W  reasons=0x{reasons:x}", flush=True)
        k += 1


if __name__ == "__main__":
    main()
