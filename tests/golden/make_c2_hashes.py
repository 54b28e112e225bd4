"""Golden fixture: entry count and an order-independent 64-bit hash of every
angle block of the C2 system matrix (BASELINE.json configs[2]), computed from
the UNMODIFIED reference compiled with the correctly rounded libm
(oracle/_ref/libctsm_ref_cr.so via detail::angle_block_entries). The GPU test
tests/test_gpu_parity_scale.py::test_c2_full_matrix_hashes builds the whole
matrix (4.6 G entries) and compares all 360 blocks bit for bit through these.

    python tests/golden/make_c2_hashes.py        # ~20 min on 8 cores

hash(block) = sum over entries of
    (bits(w) * K1) xor (((raster << 32) | column) * K2)   (mod 2^64)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402
from paper_2511_12235_b200 import CONFIGS  # noqa: E402

K1 = np.uint64(0x9E3779B97F4A7C15)
K2 = np.uint64(0xC2B2AE3D27D4EB4F)


def block_hash(raster, col, w):
    key = (raster.astype(np.uint64) << np.uint64(32)) | col.astype(np.uint64)
    with np.errstate(over="ignore"):
        m = (w.view(np.uint64) * K1) ^ (key * K2)
        return int(np.sum(m, dtype=np.uint64)), int(raster.size)


def main():
    variant = sys.argv[1] if len(sys.argv) > 1 else "ref_cr"
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
    g = CONFIGS[cfg]
    o = pyoracle.load(variant)
    threads = os.cpu_count() or 1
    h = np.zeros(g.n_angles, np.uint64)
    n = np.zeros(g.n_angles, np.int64)
    for ip in range(g.n_angles):
        r, c, w = o.angle_block_entries(g, ip, threads=threads)
        hv, nv = block_hash(r, c, w)
        h[ip], n[ip] = np.uint64(hv), nv
        if ip % 20 == 0:
            print(ip, nv, hex(hv), flush=True)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{cfg}_block_hashes_{variant}.npz")
    np.savez_compressed(out, hash=h, nnz=n)
    print("wrote", out, int(n.sum()))


if __name__ == "__main__":
    main()
