"""numpy's Generator(PCG64) draws used by the bandit, restated (test infrastructure only).

Third-party dependency: numpy 2.3.5 (``numpy/random/src/pcg64/pcg64.h``,
``numpy/random/src/distributions/distributions.c``); the reference draws
through it at colbandit/bandit.py:193 (seeding), 163-165 (warm-up
``integers(T)``), 314-315 (``random()`` then ``integers(len(un))``).

Published algorithm (PCG64 = "XSL RR 128/64" LCG; O'Neill 2014):

* state step: ``s = s * 0x2360ED051FC65DA44385DF649FCCF645 + inc (mod 2^128)``,
  output from the *advanced* state: ``rotr64(hi ^ lo, s >> 122)``;
* ``next32``: half-word buffer — if a buffered high half exists, return it;
  otherwise draw 64 bits, return the low half and buffer the high half;
* ``random()`` = ``(next64 >> 11) * 2^-53``;
* ``integers(n)`` (n <= 2^32): Lemire's nearly-divisionless bounded draw on
  ``next32``: ``m = next32 * n``; if ``(m mod 2^32) < n``, redraw while it is
  below ``(2^32 - n) mod n``; result ``m >> 32``. No draw at all when n == 1.

Seeding (SeedSequence hashing of int/tuple seeds) is not restated: both the
product and this oracle take the post-seeding state from
``np.random.default_rng(seed).bit_generator.state``.
"""

from __future__ import annotations

import numpy as np

MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1


class PCG64Ref:
    def __init__(self, state: int, inc: int, has_uint32: int = 0, uinteger: int = 0):
        self.state = state & MASK128
        self.inc = inc & MASK128
        self.has_uint32 = int(has_uint32)
        self.uinteger = int(uinteger) & 0xFFFFFFFF

    @classmethod
    def from_seed(cls, seed) -> "PCG64Ref":
        st = np.random.default_rng(seed).bit_generator.state
        return cls(st["state"]["state"], st["state"]["inc"], st["has_uint32"], st["uinteger"])

    def next64(self) -> int:
        self.state = (self.state * MULT + self.inc) & MASK128
        hi, lo = self.state >> 64, self.state & MASK64
        x = hi ^ lo
        rot = self.state >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next32(self) -> int:
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        x = self.next64()
        self.has_uint32 = 1
        self.uinteger = x >> 32
        return x & 0xFFFFFFFF

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def integers(self, n: int) -> int:
        if n < 1:
            raise ValueError("n must be >= 1")
        if n == 1:
            return 0
        m = self.next32() * n
        low = m & 0xFFFFFFFF
        if low < n:
            thr = ((1 << 32) - n) % n
            while low < thr:
                m = self.next32() * n
                low = m & 0xFFFFFFFF
        return m >> 32
