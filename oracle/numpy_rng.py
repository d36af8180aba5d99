"""Pure-Python restatement of numpy's Generator draws used by the reference's workload
generator (pkg/src/timewarp/workload.py:129-137). TEST INFRASTRUCTURE ONLY: it checks
our reading of numpy 2.x's algorithms (the basis of csrc/workload.cu) against numpy
itself; the product never imports it.

  PCG64 (XSL-RR 128/64)  numpy/random/src/pcg64/pcg64.h: pcg_setseq_128_xsl_rr_64
  next_uint32 buffering  numpy/random/_pcg64.pyx / pcg64.h: pcg64_next32
  exponential            numpy/random/src/distributions/distributions.c:
                         random_standard_exponential (+ _unlikely), ziggurat tables
  integers               numpy/random/src/distributions/distributions.c:
                         random_bounded_uint64 -> buffered_bounded_lemire_uint32
"""

from __future__ import annotations

import math

M128 = (1 << 128) - 1
MULT = (0x2360ED051FC65DA4 << 64) | 0x4385DF649FCCF645
ZIG_EXP_R = 7.69711747013104972


class Pcg64:
    def __init__(self, bitgen_state: dict) -> None:
        self.s = int(bitgen_state["state"]["state"])
        self.inc = int(bitgen_state["state"]["inc"])
        self.has32 = int(bitgen_state["has_uint32"])
        self.u32 = int(bitgen_state["uinteger"])

    def next64(self) -> int:
        self.s = (self.s * MULT + self.inc) & M128
        x = (self.s >> 64) ^ (self.s & ((1 << 64) - 1))
        rot = self.s >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)

    def next32(self) -> int:
        if self.has32:
            self.has32 = 0
            return self.u32
        n = self.next64()
        self.has32, self.u32 = 1, n >> 32
        return n & 0xFFFFFFFF

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def standard_exponential(g: Pcg64, ke, we, fe) -> float:
    while True:
        ri = g.next64() >> 3
        idx = ri & 0xFF
        ri >>= 8
        x = ri * we[idx]
        if ri < ke[idx]:
            return x
        if idx == 0:
            return ZIG_EXP_R - math.log1p(-g.next_double())
        if (fe[idx - 1] - fe[idx]) * g.next_double() + fe[idx] < math.exp(-x):
            return x


def integers_closed(g: Pcg64, low: int, high: int) -> int:
    """Generator.integers(low, high + 1) for int64 with high - low < 2^32."""
    rng = high - low
    if rng == 0:
        return low
    if rng == 0xFFFFFFFF:
        return low + g.next32()
    excl = rng + 1
    m = g.next32() * excl
    left = m & 0xFFFFFFFF
    if left < excl:
        threshold = (0xFFFFFFFF - rng) % excl
        while left < threshold:
            m = g.next32() * excl
            left = m & 0xFFFFFFFF
    return low + (m >> 32)
