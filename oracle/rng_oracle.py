"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY -- numpy's seeded normal stream.

The reference's power iterations start from
`np.random.default_rng(seed).standard_normal(n)`, masked and normalised
(fea.py:289-292; solvers.py:352-355).  The algorithm lives in numpy (a
dependency the reference pins only as numpy>=1.24, pyproject.toml:10-15; this
image has numpy 2.3): PCG64 (XSL-RR 128/64) seeded through SeedSequence, and
the 256-layer ziggurat of `random_standard_normal`
(numpy/random/src/distributions/distributions.c).  This module restates both
so that the CUDA generator (csrc/rng.cu) can be checked piece by piece:

* `pcg64_state(seed)`: the 128-bit state and increment after seeding (taken
  from numpy's own SeedSequence -- the seeding hash is not restated);
* `pcg64_raw(state, inc, n)`: the 64-bit outputs (state <- state*M + inc,
  output rotr64(hi ^ lo, hi >> 58));
* `standard_normal(seed, n, tables)`: the ziggurat over that stream;
* `read_tables(header)`: the constants from the generated CUDA header
  (tools/gen_ziggurat_tables.py), so the committed header is what is pinned.

Pinned against numpy itself: tests/test_rng.py checks `standard_normal`
bit for bit against `default_rng(seed).standard_normal` for several seeds.
"""
from __future__ import annotations

import math
import re

import numpy as np

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828


def pcg64_state(seed: int) -> tuple[int, int]:
    st = np.random.PCG64(np.random.SeedSequence(seed)).state["state"]
    return int(st["state"]), int(st["inc"])


def pcg64_raw(state: int, inc: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    for i in range(n):
        state = (state * PCG_MULT + inc) & MASK128
        hi, lo = state >> 64, state & ((1 << 64) - 1)
        x, rot = hi ^ lo, hi >> 58
        out[i] = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
    return out


def pcg64_advance(state: int, inc: int, delta: int) -> int:
    """state after `delta` steps (pcg_advance_lcg_128: O(log delta))."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, PCG_MULT, inc
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        delta >>= 1
    return (acc_mult * state + acc_plus) & MASK128


def _next_double(r) -> float:
    return float(int(r) >> 11) * (1.0 / 9007199254740992.0)


def standard_normal(seed: int, n: int, tables, raw: np.ndarray | None = None) -> np.ndarray:
    """random_standard_normal over the seeded PCG64 stream, n values."""
    ki, wi, fi = tables
    if raw is None:
        raw = np.random.PCG64(np.random.SeedSequence(seed)).random_raw(int(n * 1.05) + 256)
    idx = (raw & np.uint64(0xFF)).astype(np.int64)
    r = raw >> np.uint64(8)
    sign = (r & np.uint64(1)).astype(bool)
    rabs = (r >> np.uint64(1)) & np.uint64(0x000FFFFFFFFFFFFF)
    x = rabs.astype(np.float64) * wi[idx]
    x = np.where(sign, -x, x)
    acc = rabs < ki[idx]
    out = np.empty(n)
    j = k = 0
    while k < n:
        if acc[j]:  # 99% of attempts: one draw
            run = j
            while run < len(acc) and acc[run] and k + (run - j) < n:
                run += 1
            m = run - j
            out[k:k + m] = x[j:run]
            k += m
            j = run
            continue
        i, xj, rb = int(idx[j]), float(x[j]), int(rabs[j])
        j += 1
        if i == 0:  # tail beyond r
            while True:
                xx = -ZIG_INV_R * math.log1p(-_next_double(raw[j]))
                yy = -math.log1p(-_next_double(raw[j + 1]))
                j += 2
                if yy + yy > xx * xx:
                    out[k] = -(ZIG_R + xx) if (rb >> 8) & 1 else ZIG_R + xx
                    k += 1
                    break
        else:  # wedge
            u = _next_double(raw[j])
            j += 1
            if (fi[i - 1] - fi[i]) * u + fi[i] < math.exp(-0.5 * xj * xj):
                out[k] = xj
                k += 1
    return out


def read_tables(header: str):
    """(ki, wi, fi) from the generated csrc/ziggurat_tables.cuh."""
    text = open(header).read()

    def body(name):
        return text[text.index(f"{name}[256] = {{"):].split("};", 1)[0].split("{", 1)[1]

    ki = np.array([int(t, 16) for t in re.findall(r"0x([0-9A-F]+)ull", body("ki"))], np.uint64)
    wi = np.array([float.fromhex(t) for t in re.findall(r"[-+0-9a-fx.p]+", body("wi")) if "x" in t])
    fi = np.array([float.fromhex(t) for t in re.findall(r"[-+0-9a-fx.p]+", body("fi")) if "x" in t])
    assert ki.size == wi.size == fi.size == 256
    return ki, wi, fi


def start_vector(seed: int, fixed: np.ndarray) -> np.ndarray:
    """fea.py:289-292: masked, normalised seeded normal vector."""
    x = np.random.default_rng(seed).standard_normal(fixed.size)
    x[fixed] = 0.0
    return x / np.linalg.norm(x)
