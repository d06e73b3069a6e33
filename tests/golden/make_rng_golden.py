"""Writes rng_u32_keys.txt from rng_ref.py (plain Python ints, independent of
oracle/).  Run: python tests/golden/make_rng_golden.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import rng_ref  # noqa: E402

CASES = [(0, 0, 1, 0, 0), (0, 0, 1, 0, 1), (0, 0, 1, 0, 2), (0, 0, 1, 0, 3), (0, 0, 1, 0, 16), (0, 0, 1, 0, 47),
         (0, 0, 1, 1, 0), (0, 0, 1, 255, 16), (0, 0, 2, 0, 0), (0, 1, 1, 0, 0), (1, 0, 1, 0, 0),
         (1, 7, 300, 4095, 79), (6, 302, 17, 127, 2), (12345678901, 63, 200, 2047, 16), (2 ** 63 + 5, 5, 9, 4096, 3)]

if __name__ == "__main__":
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rng_u32_keys.txt")
    with open(path, "w") as f:
        f.write("# u32 of the composed training RNG key (DESIGN.md R13; SURVEY.md 8(c) A13), written by\n"
                "# tests/golden/make_rng_golden.py from rng_ref.py (plain Python ints, no oracle/ import).\n"
                "# columns: seed obj t ray stream u32(hex)\n")
        for (seed, obj, t, ray, stream) in CASES:
            f.write(f"{seed} {obj} {t} {ray} {stream} {rng_ref.key_u32(seed, obj, t, ray, stream):08x}\n")
    print("wrote", path)
