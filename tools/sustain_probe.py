"""How a kernel's per-launch time evolves under sustained back-to-back load
(the bench's settle-then-time protocol vs a short burst), next to a plain
device-to-device copy of the same bytes, with the SM / memory clocks and
power sampled by nvidia-smi every 50 ms.  One JSON line per kernel.

  python tools/sustain_probe.py [--seconds 3] [--window 20]
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def smi_start():
    fd, path = tempfile.mkstemp(suffix=".csv")
    os.close(fd)
    f = open(path, "w")
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,"
                          "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,temperature.gpu,"
                          "temperature.memory", "--format=csv,noheader,nounits", "-lms", "50", "-i", "0"],
                         stdout=f, stderr=subprocess.DEVNULL)
    return p, f, path


def smi_stop(h):
    p, f, path = h
    p.terminate()
    p.wait()
    f.close()
    rows = [l.strip().split(", ") for l in open(path) if l.strip()]
    os.unlink(path)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--window", type=int, default=20)
    a = ap.parse_args()
    import torch
    import iqsynth
    from iqsynth import dist as D
    import paper_2603_28430_b200 as iq
    n = 1 << 20
    cases = []
    for dt, tdt, bits in (("f16", torch.float16, 3), ("f32", torch.float32, 3), ("f16", torch.float16, 2)):
        xs, _, _ = D.rank_buffers(2, n, 128, tdt, "cuda", buffers=2)
        ys = [torch.empty_like(x) for x in xs]
        p = iq.iq_make_params(128, bits, iq.FULL, iqsynth.PARAMS_SEED, device=0)
        cases.append((f"roundtrip_{dt}_b{bits}", lambda i, p=p, xs=xs, ys=ys: iq.iq_roundtrip(p, xs[i & 1], y=ys[i & 1]),
                      2 * n * 128 * (2 if dt == "f16" else 4)))
        if bits == 3:
            cases.append((f"copy_{dt}", lambda i, xs=xs, ys=ys: ys[i & 1].copy_(xs[i & 1]),
                          2 * n * 128 * (2 if dt == "f16" else 4)))
    for name, fn, nbytes in cases:
        torch.cuda.synchronize()
        time.sleep(1.0)                                # let the clocks recover between cases
        h = smi_start()
        time.sleep(0.2)
        evs = []
        t0 = time.time()
        i = 0
        while time.time() - t0 < a.seconds:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            evs.append(e)
            for _ in range(a.window):
                fn(i)
                i += 1
            if len(evs) % 8 == 0:
                torch.cuda.synchronize()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        evs.append(e)
        torch.cuda.synchronize()
        rows = smi_stop(h)
        us = [evs[k].elapsed_time(evs[k + 1]) * 1e3 / a.window for k in range(len(evs) - 1)]
        pick = [0, 1, 2, 5, 10, 20, 50, 100, 200, 400, len(us) // 2, len(us) - 1]
        series = {k: round(us[k], 1) for k in pick if k < len(us)}
        sm = [float(r[1]) for r in rows if len(r) > 3 and r[1].replace('.', '').isdigit()]
        mem = [float(r[2]) for r in rows if len(r) > 3 and r[2].replace('.', '').isdigit()]
        pw = [float(r[3]) for r in rows if len(r) > 3 and r[3].replace('.', '').isdigit()]
        cap = sum(1 for r in rows if len(r) > 4 and r[4] == "Active")
        print(json.dumps({"kernel": name, "launches": i, "us_window_index_to_us": series,
                          "first_window_us": round(us[0], 1), "median_us": round(sorted(us)[len(us) // 2], 1),
                          "last_window_us": round(us[-1], 1),
                          "GB/s_first": nbytes / us[0] / 1e3, "GB/s_median": nbytes / sorted(us)[len(us) // 2] / 1e3,
                          "sm_mhz": [min(sm or [0]), sorted(sm or [0])[len(sm or [0]) // 2], max(sm or [0])],
                          "mem_mhz": [min(mem or [0]), max(mem or [0])], "power_w_max": max(pw or [0]),
                          "power_w_median": sorted(pw or [0])[len(pw or [0]) // 2],
                          "sw_power_cap_samples": cap, "samples": len(rows)}), flush=True)


if __name__ == "__main__":
    main()
