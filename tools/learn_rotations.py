"""Learn IsoQuant block rotations on the GPU (PAPER.md "Parameterization and
Learning"; R29/R30) — an example of the learning API.

Each step: iq_distortion_grad (one kernel: dL/dM per block of the normalised
stage-1 distortion) -> iq_rot_grad_from_operator_grad (host chain rule to the
unit quaternions / angles, tangent-projected) -> a normalised gradient step
-> iq_make_params_explicit (renormalises q = u / ||u||).  Prints the
distortion per step and the roundtrip MSE before and after.

  python tools/learn_rotations.py [--d 128 --bits 2 --variant full --rows 65536 --steps 30 --lr 0.05]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--bits", type=int, default=2)
    ap.add_argument("--variant", default="full")
    ap.add_argument("--rows", type=int, default=1 << 16)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--lr", type=float, default=0.05)
    a = ap.parse_args()
    import numpy as np
    import torch
    import iqsynth
    import paper_2603_28430_b200 as iq

    v = iq.VARIANTS[a.variant]
    # unequal per-coordinate energy: the case the rotation is for
    X = torch.from_numpy(iqsynth.outlier_vectors(a.rows, a.d, 7, np.float32)).cuda()
    p = iq.iq_make_params(a.d, a.bits, v, iqsynth.PARAMS_SEED, device=0)
    rot = iq.iq_export_params(p)["rot"]
    n_units = rot.size // (2 if v == iq.PLANAR2D else 4)

    def mse(params):
        y = iq.iq_roundtrip(params, X)
        return float(((X - y) ** 2).mean())

    m0 = mse(p)
    for step in range(a.steps):
        grad, loss = iq.iq_distortion_grad(p, X)
        g = iq.iq_rot_grad_from_operator_grad(p, grad.cpu().numpy())
        print(f"step {step:3d}  distortion {float(loss):.6e}", flush=True)
        rot = rot - a.lr * np.sqrt(n_units) * g / max(np.linalg.norm(g), 1e-30)
        p = iq.iq_make_params_explicit(a.d, a.bits, v, rot, device=0)
    print(f"roundtrip MSE: random rotations {m0:.6e} -> learned {mse(p):.6e}")


if __name__ == "__main__":
    main()
