"""Load the committed golden fixtures (tests/golden/*.npz, made by
oracle/make_golden.py) into plain float arrays."""

import glob
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def bf16_bits_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")) as z:
        g = {k: z[k] for k in z.files}
    g["dtype"] = str(g["dtype"])
    g["source"] = str(g["source"])
    g["compensator"] = str(g["compensator"])
    g["grid"] = tuple(int(a) for a in g["grid"])
    g["split"] = tuple(int(a) for a in g["split"])
    g["block3"] = tuple(int(a) for a in g["block3"])
    g["topk"] = int(g["topk"])
    g["keep"] = float(g["keep"])
    g["use_pe"] = bool(g["use_pe"])
    if g["dtype"] == "bf16":
        for n in ("q", "k", "v", "x"):
            g[n] = bf16_bits_to_f32(g[n])
    return g
