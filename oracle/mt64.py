"""ORACLE ONLY — std::mt19937_64 (the C++11 standard's 64-bit Mersenne
Twister, the generator every seeded stream in the reference uses), restated
from its published parameters so oracle/lstm.py can reproduce the
reference's θ initialisation (src/lstm.cpp:77-81) bit for bit."""
from __future__ import annotations

_MASK = (1 << 64) - 1
_NN, _MM = 312, 156
_MATRIX_A = 0xB5026F5AA96619E9
_UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF


class MT19937_64:
    def __init__(self, seed: int):
        mt = [0] * _NN
        mt[0] = seed & _MASK
        for i in range(1, _NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self.mt, self.i = mt, _NN

    def _twist(self):
        mt = self.mt
        for i in range(_NN):
            x = (mt[i] & _UM) | (mt[(i + 1) % _NN] & _LM)
            xa = x >> 1
            if x & 1:
                xa ^= _MATRIX_A
            mt[i] = mt[(i + _MM) % _NN] ^ xa
        self.i = 0

    def next(self) -> int:
        if self.i >= _NN:
            self._twist()
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _MASK
