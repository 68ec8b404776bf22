"""Feature-noise restatement -- TEST INFRASTRUCTURE ONLY (only tests/ and
tools/ import this module; the product package never does).

extract_feature (reference classifiers.py:152-158) draws
default_rng([seed, oid, 1]).standard_normal(D): numpy 2.3.5's
random_standard_normal (numpy/random/src/distributions/distributions.c, a
256-layer ziggurat over PCG64 next_uint64 / next_double) whose slow paths call
glibc's log1p (npy_log1p) and exp.  This module restates:

* `normals(raw, n)`: the ziggurat over a sequence of raw PCG64 words, with the
  tables read from the committed header csrc/ziggurat_tables.cuh (which
  tools/gen_ziggurat.py extracted from numpy's extension module);
* `glibc_log1p(x)`: glibc 2.39's x86_64 __log1p_fma (the ifunc the image's
  CPUs run), i.e. fdlibm s_log1p.c with the fused multiply-adds GCC emitted
  under -mfma, transcribed from the shipped machine code -- the restatement
  csrc/noise.cu runs on the device.

Pinned by tests/test_noise_restatement.py: `normals` == Generator.standard_normal
and `glibc_log1p` == math.log1p (both the real libraries), bit for bit.
"""

from __future__ import annotations

import math
import os
import re
import struct
from fractions import Fraction

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "paper_1801_03493_b200", "csrc", "ziggurat_tables.cuh")
ZR = 3.6541528853610087963519472518       # ziggurat_nor_r
ZINV = 0.27366123732975827203338247596    # ziggurat_nor_inv_r


def header_tables(path: str = HEADER):
    """(ki uint64[256], wi float64[256], fi float64[256]) from the header."""
    txt = open(path).read()
    out = []
    for name in ("kZigKi", "kZigWi", "kZigFi"):
        body = txt.split(name + "[256] = {", 1)[1].split("};", 1)[0]
        vals = np.array([int(v, 16) for v in re.findall(r"0x([0-9a-f]+)ull", body)], np.uint64)
        assert vals.size == 256, name
        out.append(vals)
    return out[0], out[1].view(np.float64), out[2].view(np.float64)


def normals(raw, n: int, tables=None, log1p=math.log1p, exp=math.exp) -> np.ndarray:
    """random_standard_normal (distributions.c) n times over raw PCG64 words."""
    ki, wi, fi = header_tables() if tables is None else tables
    out, it = [], iter(raw)
    nxt = lambda: int(next(it))
    nd = lambda: (nxt() >> 11) * (1.0 / 9007199254740992.0)
    while len(out) < n:
        while True:
            r = nxt()
            idx = r & 0xff
            r >>= 8
            rabs = (r >> 1) & 0x000fffffffffffff
            x = rabs * float(wi[idx])
            if r & 1:
                x = -x
            if rabs < int(ki[idx]):
                out.append(x)
                break
            if idx == 0:
                while True:
                    xx = -ZINV * log1p(-nd())
                    yy = -log1p(-nd())
                    if yy + yy > xx * xx:
                        out.append(-(ZR + xx) if ((rabs >> 8) & 1) else ZR + xx)
                        break
                break
            if (float(fi[idx - 1]) - float(fi[idx])) * nd() + float(fi[idx]) < exp(-0.5 * x * x):
                out.append(x)
                break
    return np.array(out)


def _fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _hi(x: float) -> int:
    v = struct.unpack("<Q", struct.pack("<d", x))[0] >> 32
    return v - (1 << 32) if v >= (1 << 31) else v


def _set_hi(x: float, h: int) -> float:
    b = struct.unpack("<Q", struct.pack("<d", x))[0]
    return struct.unpack("<d", struct.pack("<Q", ((h & 0xffffffff) << 32) | (b & 0xffffffff)))[0]


_LN2_HI, _LN2_LO = 6.93147180369123816490e-01, 1.90821492927058770002e-10
_LP = (0.0, 6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01, 2.222219843214978396e-01,
       1.818357216161805012e-01, 1.531383769920937332e-01, 1.479819860511658591e-01)


def glibc_log1p(x: float) -> float:
    """glibc 2.39 __log1p_fma for finite x > -1 (csrc/noise.cu glibc_log1p)."""
    hx = _hi(x)
    ax = hx & 0x7fffffff
    k, hu, f, c = 1, 0, 0.0, 0.0
    if hx < 0x3FDA827A:
        if ax >= 0x3ff00000:
            raise ValueError("x <= -1")
        if ax < 0x3e200000:
            return x if ax < 0x3c900000 else _fma(-(x * x), 0.5, x)
        if hx > 0 or hx <= _hi(struct.unpack("<d", struct.pack("<Q", 0xbfd2bec3 << 32))[0]):
            k, f, hu = 0, x, 1
    if k != 0:
        u = x + 1.0
        hu = _hi(u)
        k = (hu >> 20) - 1023
        c = (1.0 - (u - x)) if k > 0 else (x - (u - 1.0))
        c /= u
        hu &= 0x000fffff
        if hu < 0x6a09e:
            u = _set_hi(u, hu | 0x3ff00000)
        else:
            k += 1
            u = _set_hi(u, hu | 0x3fe00000)
            hu = (0x00100000 - hu) >> 2
        f = u - 1.0
    hfsq = (f * 0.5) * f
    if hu == 0:
        if f == 0.0:
            return 0.0 if k == 0 else _fma(k, _LN2_HI, _fma(k, _LN2_LO, c))
        R = _fma(-f, 0.6666666666666666, 1.0) * hfsq
        return f - R if k == 0 else _fma(k, _LN2_HI, -((R - _fma(k, _LN2_LO, c)) - f))
    s = f / (f + 2.0)
    z = s * s
    R2, R3, R4 = _fma(z, _LP[3], _LP[2]), _fma(z, _LP[5], _LP[4]), _fma(z, _LP[7], _LP[6])
    z2 = z * z
    z4 = z2 * z2
    z6 = z2 * z4
    t = _fma(z4, R3, _fma(z, _LP[1], z2 * R2))
    w = (_fma(z6, R4, t) + hfsq) * s
    if k == 0:
        return f - (hfsq - w)
    return _fma(k, _LN2_HI, -((hfsq - (_fma(k, _LN2_LO, c) + w)) - f))
