"""Seed tree and numpy-PCG64 stream semantics (oracle; test infrastructure only).

Reference: ``src/rng.py:15-26`` (child_seed / make_rng).  The streams
themselves are numpy 2.3.5 ``Generator(PCG64(seed))``; ``PCG64Emu`` is an
integer-exact restatement of the numpy algorithms the reference calls
(SeedSequence hash mixing, PCG64 XSL-RR, the persistent 32-bit half buffer,
Lemire bounded ints, masked-rejection Fisher-Yates, ``choice(p=)``), kept
pure-Python so the CUDA port (``csrc/rng.cuh``) can be checked against it
draw-for-draw in ``tests/test_rng_emu.py``.
"""

import hashlib

import numpy as np

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1
M128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def child_seed(parent, *labels):
    """SHA-256 child seed; mirrors ``src/rng.py:15-19``."""
    text = str(int(parent) & M64)
    for lab in labels:
        text += ":" + str(lab)
    return int.from_bytes(hashlib.sha256(text.encode("utf-8")).digest()[:8], "little")


def make_rng(seed, *labels):
    """numpy Generator for (seed, labels); mirrors ``src/rng.py:22-26``."""
    if labels:
        seed = child_seed(seed, *labels)
    return np.random.Generator(np.random.PCG64(int(seed) & M64))


# -- SeedSequence (numpy/random/bit_generator.pyx) -----------------------------

_INIT_A, _MULT_A = 0x43B0D7E5, 0x931E8875
_INIT_B, _MULT_B = 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715


def _words32(value):
    value = int(value)
    if value == 0:
        return [0]
    out = []
    while value:
        out.append(value & M32)
        value >>= 32
    return out


def seed_sequence_words(entropy, n_words32=8):
    """``SeedSequence(entropy).generate_state(n_words32//2, uint64)`` as uint32 words."""
    ent = _words32(entropy)
    hc = [_INIT_A]

    def hashmix(v):
        v = (v ^ hc[0]) & M32
        hc[0] = (hc[0] * _MULT_A) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (_MIX_L * x - _MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    out = []
    h = _INIT_B
    for i in range(n_words32):
        v = pool[i % 4] ^ h
        h = (h * _MULT_B) & M32
        v = (v * h) & M32
        out.append(v ^ (v >> 16))
    return out


class PCG64Emu:
    """numpy ``Generator(PCG64(seed))`` restated on Python ints."""

    def __init__(self, seed):
        w = seed_sequence_words(seed, 8)
        v = [w[2 * i] | (w[2 * i + 1] << 32) for i in range(4)]
        initstate = (v[0] << 64) | v[1]
        initseq = (v[2] << 64) | v[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & M128
        self._step()
        self.has32 = False
        self.buf32 = 0

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self):
        self._step()
        hi, lo = self.state >> 64, self.state & M64
        x = hi ^ lo
        rot = hi >> 58
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next32(self):
        if self.has32:
            self.has32 = False
            return self.buf32
        v = self.next64()
        self.has32 = True
        self.buf32 = v >> 32
        return v & M32

    def random(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def uniform(self, lo, hi):
        span = float(hi) - float(lo)
        return float(lo) + span * self.random()

    def integers(self, lo, hi=None):
        """``Generator.integers(lo, hi)`` (int64, endpoint=False)."""
        if hi is None:
            lo, hi = 0, lo
        rng = hi - lo - 1
        if rng == 0:
            return lo
        if rng < M32:
            excl = rng + 1
            m = self.next32() * excl
            left = m & M32
            if left < excl:
                thr = (M32 - rng) % excl
                while left < thr:
                    m = self.next32() * excl
                    left = m & M32
            return lo + (m >> 32)
        if rng == M32:
            return lo + self.next32()
        excl = rng + 1
        m = self.next64() * excl
        left = m & M64
        if left < excl:
            thr = (M64 - rng) % excl
            while left < thr:
                m = self.next64() * excl
                left = m & M64
        return lo + (m >> 64)

    def interval(self, mx):
        """numpy ``random_interval(bitgen, max)``."""
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= M32:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    def permutation(self, n):
        a = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            a[i], a[j] = a[j], a[i]
        return a

    def choice_p(self, p):
        """``Generator.choice(len(p), p=p)`` for a float64 vector p."""
        cdf = np.cumsum(np.asarray(p, dtype=np.float64))
        cdf = cdf / cdf[-1]
        u = self.random()
        return int(np.searchsorted(cdf, u, side="right"))


def pairwise_sum(vals):
    """numpy float64 pairwise summation of a 1-D contiguous vector (n <= 128)."""
    a = [float(v) for v in vals]
    n = len(a)
    if n < 8:
        res = 0.0
        for v in a:
            res += v
        return res
    r = a[:8]
    i = 8
    while i < n - (n % 8):
        for k in range(8):
            r[k] += a[i + k]
        i += 8
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    while i < n:
        res += a[i]
        i += 1
    return res
