"""Pure-Python restatement of numpy's PCG64 bit generator (test oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

numpy's `PCG64` is PCG-XSL-RR 128/64 ("setseq" variant): a 128-bit LCG
    s <- s * MULT + inc   (mod 2**128)
followed by the XSL-RR output of the *new* state:
    x = hi64(s) ^ lo64(s);  out = rotr64(x, s >> 122).
`Generator.random()` maps one 64-bit output to (out >> 11) * 2**-53.
The reference draws sampler priorities with exactly that call
(`gnnio/sampler.py:90`, stream from `default_rng((cfg.seed, batch_seed))`
at `sampler.py:61-62`). Jump-ahead is the standard LCG power-by-squaring.

The initial (state, inc) of a stream is taken from numpy itself
(`default_rng(...).bit_generator.state`), so SeedSequence hashing is never
re-implemented; this module only restates the stepping arithmetic.
"""

from __future__ import annotations

import numpy as np

MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1
MULT = (2549297995355413924 << 64) + 4865540595714422341


def stream_state(seed_tuple) -> tuple[int, int]:
    """(state, inc) of `np.random.default_rng(seed_tuple)` as Python ints."""
    st = np.random.default_rng(seed_tuple).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def step(state: int, inc: int) -> int:
    return (state * MULT + inc) & MASK128


def output(state: int) -> int:
    hi, lo = state >> 64, state & MASK64
    x = hi ^ lo
    rot = state >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64


def advance(state: int, inc: int, delta: int) -> int:
    """State after `delta` LCG steps (power-by-squaring)."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = MULT, inc
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        delta >>= 1
    return (acc_mult * state + acc_plus) & MASK128


def draw_u53(state: int, inc: int, index: int) -> int:
    """53-bit integer m of the `index`-th `Generator.random()` draw (0-based)
    of the stream; the double is m * 2**-53."""
    s = advance(state, inc, index + 1)
    return output(s) >> 11


def affine_map(inc: int, delta: int) -> tuple[int, int]:
    """(A, C) with s -> A*s + C advancing `delta` steps."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = MULT, inc
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        delta >>= 1
    return acc_mult, acc_plus


TABLE_ROWS = 1 + 16 * 15


def jump_table(state: int, inc: int) -> np.ndarray:
    """[241, 4] uint64 rows. Row 0 = (state_hi, state_lo, inc_hi, inc_lo);
    row 1 + 15*i + (j-1) = (A_hi, A_lo, C_hi, C_lo) with s -> A*s + C
    advancing j * 16**i steps. Same layout the CUDA kernel `bgl_pcg64_tables`
    produces (a jump is one map per nonzero hex digit)."""
    rows = [(state >> 64, state & MASK64, inc >> 64, inc & MASK64)]
    for i in range(16):
        for j in range(1, 16):
            a, c = affine_map(inc, j * 16 ** i)
            rows.append((a >> 64, a & MASK64, c >> 64, c & MASK64))
    return np.array(rows, dtype=np.uint64)
