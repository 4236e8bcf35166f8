"""Design check for the GPU Gaussian generator (K0): a vectorized numpy
re-implementation of numpy's Generator(Philox(key)).standard_normal as a
*parallel* algorithm (every stream position evaluated independently, then a
sparse fix-up of the rare rejection positions), compared bit-for-bit with
numpy.  Also dumps the ziggurat tables into the CUDA header the kernel uses.

Usage: python tools/philox_ziggurat.py [--emit-header]
"""
import math
import os
import struct
import sys

import numpy as np

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def tables():
    d = os.path.dirname(np.__file__)
    lib = [f for f in os.listdir(d + "/random") if f.startswith("_generator") and f.endswith(".so")][0]
    b = open(os.path.join(d, "random", lib), "rb").read()
    off = b.find(struct.pack("<d", 9.77101701267671596263e-01)) - 8
    fi = np.frombuffer(b, dtype="<f8", count=256, offset=off).copy()
    wi = np.frombuffer(b, dtype="<f8", count=256, offset=off + 2048).copy()
    ki = np.frombuffer(b, dtype="<u8", count=256, offset=off + 4096).copy()
    return ki, wi, fi


def mulhilo(a, m):
    a = a.astype(np.uint64)
    m = np.uint64(m)
    lo = a * m
    a0, a1 = a & np.uint64(0xFFFFFFFF), a >> np.uint64(32)
    m0, m1 = m & np.uint64(0xFFFFFFFF), m >> np.uint64(32)
    p00, p01, p10, p11 = a0 * m0, a0 * m1, a1 * m0, a1 * m1
    mid = (p00 >> np.uint64(32)) + (p01 & np.uint64(0xFFFFFFFF)) + (p10 & np.uint64(0xFFFFFFFF))
    hi = p11 + (p01 >> np.uint64(32)) + (p10 >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, lo


def philox_blocks(ctr0, key):
    """4x64-10 for counters ctr0 (array, upper counter words 0)."""
    c = [ctr0.astype(np.uint64), np.zeros_like(ctr0, dtype=np.uint64),
         np.zeros_like(ctr0, dtype=np.uint64), np.zeros_like(ctr0, dtype=np.uint64)]
    k0, k1 = np.uint64(key[0]), np.uint64(key[1])
    with np.errstate(over="ignore"):
        for _ in range(10):
            hi0, lo0 = mulhilo(c[0], M0)
            hi1, lo1 = mulhilo(c[2], M1)
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
            k0 = np.uint64((int(k0) + W0) & MASK)
            k1 = np.uint64((int(k1) + W1) & MASK)
    return np.stack(c, axis=1)   # (blocks, 4)


def raw_stream(key, n):
    nb = (n + 3) // 4
    return philox_blocks(np.arange(1, nb + 1, dtype=np.uint64), key).reshape(-1)[:n]


def normals_parallel(key, count, ki, wi, fi):
    r_ = 3.6541528853610087963519472518
    inv_r = 0.27366123732975827203338247596
    L = int(count * 1.02) + 64
    while True:
        u = raw_stream(key, L + 16)
        idx = (u & np.uint64(0xFF)).astype(np.int64)
        r = u >> np.uint64(8)
        sign = (r & np.uint64(1)).astype(bool)
        rabs = (r >> np.uint64(1)) & np.uint64(0x000FFFFFFFFFFFFF)
        x = rabs.astype(np.float64) * wi[idx]
        x = np.where(sign, -x, x)
        fast = rabs < ki[idx]
        # special positions: evaluate the full attempt sequentially (rare)
        consumed = np.ones(L, dtype=np.int64)
        produce = fast[:L].copy()
        val = x[:L].copy()
        for t in np.flatnonzero(~fast[:L]):
            if idx[t] == 0:
                j = t + 1
                while True:
                    xx = -inv_r * math.log1p(-float(u[j] >> np.uint64(11)) * (1.0 / 9007199254740992.0))
                    yy = -math.log1p(-float(u[j + 1] >> np.uint64(11)) * (1.0 / 9007199254740992.0))
                    j += 2
                    if yy + yy > xx * xx:
                        val[t] = -(r_ + xx) if (int(rabs[t]) >> 8) & 1 else r_ + xx
                        break
                consumed[t] = j - t
                produce[t] = True
            else:
                nd = float(u[t + 1] >> np.uint64(11)) * (1.0 / 9007199254740992.0)
                consumed[t] = 2
                produce[t] = ((fi[idx[t] - 1] - fi[idx[t]]) * nd + fi[idx[t]]) < math.exp(-0.5 * x[t] * x[t])
        # starts: walk the special positions in order (the fix-up pass)
        start = np.ones(L, dtype=bool)
        skip = 0
        for t in np.flatnonzero(consumed > 1):
            if t < skip:
                continue
            start[t + 1:t + consumed[t]] = False
            skip = t + consumed[t]
        keep = start & produce
        out = val[keep]
        if out.size >= count:
            return out[:count]
        L *= 2


def emit_header(ki, wi, fi, path):
    with open(path, "w") as f:
        f.write("// Ziggurat tables of numpy's Generator.standard_normal (256 layers),\n"
                "// extracted by tools/philox_ziggurat.py from numpy's own binary and\n"
                "// verified bit-for-bit against numpy's output; do not edit.\n#pragma once\n"
                "#include <stdint.h>\nnamespace lr {\n")
        f.write("__constant__ uint64_t kZigKi[256] = {\n")
        f.write(",\n".join("  0x%016xULL" % int(v) for v in ki) + "};\n")
        for name, arr in (("kZigWi", wi), ("kZigFi", fi)):
            f.write(f"__constant__ double {name}[256] = {{\n")
            f.write(",\n".join("  %s" % float(v).hex() for v in arr) + "};\n")
        f.write("}  // namespace lr\n")


if __name__ == "__main__":
    ki, wi, fi = tables()
    for seed, stream, n in [(2, 0x67617573, 1_000_000), (1, 0x67617573, 61440),
                            (5, 0x70726F62, 200_000), (123456789, 0x67617573, 500_000)]:
        key = (seed, stream)
        ref = np.random.Generator(np.random.Philox(key=seed | (stream << 64))).standard_normal(n)
        got = normals_parallel(key, n, ki, wi, fi)
        diff = np.flatnonzero(ref != got)
        print(f"seed {seed} stream {stream:#x} n {n}: {diff.size} mismatches",
              ("first at %d: %r vs %r" % (diff[0], ref[diff[0]], got[diff[0]])) if diff.size else "")
    if "--emit-header" in sys.argv:
        out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "paper_0909_4061_b200", "csrc", "ziggurat_tables.cuh")
        emit_header(ki, wi, fi, out)
        print("wrote", out)
