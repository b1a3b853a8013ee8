"""Python port of the reference's deterministic RNG (rng.hpp:12-58) -- test infrastructure,
so property tests draw exactly the instances the reference's own tests draw.
Pinned against the compiled reference in tests/test_oracle_pins.py."""
M64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D4A2FA9FB8476D) & M64
    return x ^ (x >> 31)


def hash_mix(a, b):
    return splitmix64(a ^ splitmix64(b))


def hash_str(s):
    h = 0xCBF29CE484222325
    for c in s.encode():
        h = hash_mix(h, c)
    return h


class MT19937_64:
    N, M = 312, 156

    def __init__(self, seed):
        self.mt = [0] * self.N
        self.mt[0] = seed & M64
        for i in range(1, self.N):
            p = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (p ^ (p >> 62)) + i) & M64
        self.idx = self.N

    def _twist(self):
        mt = self.mt
        for i in range(self.N):
            y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % self.N] & 0x7FFFFFFF)
            v = mt[(i + self.M) % self.N] ^ (y >> 1)
            if y & 1:
                v ^= 0xB5026F5AA96619E9
            mt[i] = v
        self.idx = 0

    def __call__(self):
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M64


class Rng:
    def __init__(self, seed):
        self.eng = MT19937_64(seed)

    @staticmethod
    def substream(seed, label):
        return Rng(hash_mix(seed, hash_str(label)))

    def uniform(self):
        return (self.eng() >> 11) * (2.0 ** -53)

    def uniform_int(self, lo, hi):
        span = (hi - lo) + 1
        return lo + self.eng() % span
