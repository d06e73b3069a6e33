"""RO-MAP hot-path ORACLE -- test infrastructure, NOT product code.

A plain, slow, obviously-correct CPU implementation (numpy) of what the
B200 path computes, written from the paper (/root/reference/PAPER.md, cited as
PAPER.md:<line>) and the readings listed in DESIGN.md ("Readings").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2304_05735_b200`` + ``libromap.so``) never imports it, and it never
imports the product: the two share no code (no kernels, headers, helpers,
tables or constants).

Precision: every step that decides an integer or is required to be bit-exact
(ray generation, ray/box segment, sample distances, normalized positions,
hash indices -- BASELINE north_star) is computed in IEEE fp32 with one rounding
per operation, exactly as the method's kernel precision; everything downstream
(interpolation weights/features, MLP, volume rendering, losses, backward, Adam)
is computed in fp64.

Parity status per function is listed in ``oracle/romap_oracle.py``'s header and
in DESIGN.md ("Oracle pins").
"""
from .romap_oracle import *  # noqa: F401,F403
