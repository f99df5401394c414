"""Helpers to load the golden fixtures written by tests/golden/make_golden.py."""

import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def search_cases():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "search_*.npz")))


def logs(offsets, flat):
    return [flat[offsets[i]:offsets[i + 1]] for i in range(offsets.size - 1)]


def split_centroids(flat, sizes):
    out, pos = [], 0
    for s in sizes:
        out.append(flat[pos:pos + 256 * int(s)].reshape(256, int(s)))
        pos += 256 * int(s)
    return out
