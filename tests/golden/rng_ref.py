"""Independent reference of the training RNG key composition (R13,
SURVEY.md 8(c) A13; SPEC.md:436,456 per-object RNG streams), written with plain
Python integers from the text of the reading -- NOT from oracle/ (it imports
nothing).  Used (a) by make_rng_golden.py to write rng_u32_keys.txt and (b) by
tests/test_oracle_pins.py to pin the oracle's stream layout.

  mix(z): SplitMix64 finalizer  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9;
          z ^= z >> 27; z *= 0x94D049BB133111EB; z ^= z >> 31   (mod 2^64)
  key = mix(mix(mix(mix(seed + 0x9E3779B97F4A7C15) ^ obj) ^ t) ^ ((ray << 8) | stream))
  u32 = key >> 32;  unit = (u32 >> 8) * 2^-24;  pixel = (u32 * total) >> 32
  streams: 0 pixel, 1..3 background colour r, g, b, 16 + i jitter of sample i
"""
M64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
STREAM_PIXEL, STREAM_BG0, STREAM_JITTER0 = 0, 1, 16


def mix(z):
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def key_u32(seed, obj, t, ray, stream):
    k = mix((seed + GOLDEN_GAMMA) & M64)
    k = mix(k ^ (obj & M64))
    k = mix(k ^ (t & M64))
    k = mix(k ^ (((ray << 8) | stream) & M64))
    return k >> 32


def unit(u32):
    return (u32 >> 8) * 2.0 ** -24


def pixel_index(u32, total):
    return (u32 * total) >> 32
