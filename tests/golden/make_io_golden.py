"""Reader fixtures: PGIX graph files (valid and corrupted) with the READ-ONLY
reference reader's outcome (io.py:254-278), for the native loader's tests.

Run here (never on the GPU box -- /root/reference does not exist there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py

Writes tests/golden/io_graph_cases.npz: per case the file bytes, and either
the adjacency/degrees/medoid the reference read or the exception class name
and message (with the file path replaced by "{path}").
"""

from __future__ import annotations

import os
import struct
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

from bang import io as rio  # noqa: E402


def blob(lists, n=None, R=3, medoid=0, magic=b"PGIX", version=1, extra=b""):
    n = len(lists) if n is None else n
    b = magic + struct.pack("<4I", version, n, R, medoid)
    for ids in lists:
        b += struct.pack("<I", len(ids)) + struct.pack(f"<{len(ids)}I", *ids)
    return b + extra


def cases():
    rng = np.random.default_rng(5)
    big = []
    for i in range(500):
        ids = rng.choice(499, size=int(rng.integers(0, 9)), replace=False)
        big.append([int(v) + (v >= i) for v in ids])  # no self-loops, no duplicates
    ok = blob([[1, 2], [], [0, 1, 3], [2]], R=3, medoid=2)
    return {
        "valid": ok,
        "valid_big": blob(big, R=8, medoid=17),
        "valid_empty_graph": blob([], R=4),
        "bad_magic": b"PGIY" + ok[4:],
        "bad_version": blob([[1], [0]], version=2),
        "short_header": ok[:10],
        "degree_over_bound": blob([[1], [0, 1, 2, 0]], R=3),
        "id_out_of_range": blob([[1], [7], [0]], R=3),
        "id_range_before_truncation": blob([[1], [9]], n=4, R=3),
        "truncated_length": blob([[1], [0]], n=3, R=3),
        "truncated_ids": ok[:-2],
        "truncated_ids_mid": blob([[1, 2], [0, 2], [0, 1]], R=3)[:-4],
        "truncated_length_partial": blob([[1], [0]], n=3, R=3) + b"\0\0",
        "self_loop": blob([[0], [0]], R=3),
        "trailing_bytes": ok + b"\0\0\0\0",
        "trailing_partial_word": ok + b"\0\0",
    }


def main():
    out = {}
    names = []
    with tempfile.TemporaryDirectory() as d:
        for name, b in cases().items():
            path = os.path.join(d, name + ".pgix")
            with open(path, "wb") as f:
                f.write(b)
            names.append(name)
            out[f"{name}__bytes"] = np.frombuffer(b, np.uint8)
            try:
                g = rio.read_graph(path)
            except Exception as e:  # noqa: BLE001 -- the class is the fixture
                out[f"{name}__error"] = np.array(type(e).__name__)
                out[f"{name}__message"] = np.array(str(e).replace(path, "{path}"))
            else:
                out[f"{name}__adjacency"] = g.adjacency
                out[f"{name}__degrees"] = g.degrees
                out[f"{name}__medoid"] = np.array(g.medoid)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "io_graph_cases.npz"), **out)
    for name in names:
        print(name, out.get(f"{name}__error", "ok"), out.get(f"{name}__message", ""))


if __name__ == "__main__":
    main()
