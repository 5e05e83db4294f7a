"""Golden MC-MLP trajectory from the reference's own training loop.

Runs oracle/_ref's mcfref_mlp_train (the reference's MCSequential / MCLinear /
ReLU / cross_entropy_loss / Tape / MCSGD, compiled unmodified) on a small MLP
with config-3-style inputs and stores inputs, per-step losses and the final
MC parameters.  Run where /root/reference exists:

    python tests/golden/make_golden_mlp.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2207_08867_b200 import mlp  # noqa: E402

DIMS = [24, 32, 32, 10]
N, STEPS, LR = 48, 8, 0.01


def main():
    params = mlp.init_params(DIMS, 2, seed=3900)
    x, y = mlp.make_batch(N, DIMS[0], DIMS[-1], seed_x=3901, seed_y=3902)
    losses, final = oracle.mlp_train_reference(DIMS, 2, params, x, y, STEPS, LR)
    out = {"dims": np.array(DIMS), "x": x, "y": y, "losses": losses, "lr": np.array([LR])}
    for l, ((w, b), (wf, bf)) in enumerate(zip(params, final)):
        out[f"w{l}"], out[f"b{l}"], out[f"w{l}_final"], out[f"b{l}_final"] = w, b, wf, bf
    path = os.path.join(HERE, "golden_mlp.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes; losses", losses)


if __name__ == "__main__":
    main()
