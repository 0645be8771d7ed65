"""CPU oracle for the BGL per-mini-batch preprocessing path.

TEST INFRASTRUCTURE ONLY. Nothing in the product package
(`paper_2112_08541_b200/`) may import, call or link anything under this
directory. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline / `--impl reference` arm use it, and there only as the checker or the
timed CPU reference, never as the thing shipped.

The oracle restates, in plain numpy / Python, the algorithm of the reference
package `gnnio` (`/root/reference/pkg/src/gnnio`) for every row of SURVEY.md
§8(a). Each function cites the reference file:line it follows.

Parity pinning: the restatement is checked against golden vectors produced by
running the reference itself (`tests/golden/make_golden.py`, committed with
its outputs under `tests/golden/`), see `tests/test_oracle_golden.py`.

Third-party arithmetic the reference relies on is numpy (unpinned,
`pkg/pyproject.toml:10-12`; numpy 2.3.5 in this image):
  * `np.random.default_rng(seed)` -> SeedSequence -> PCG64 (XSL-RR 128/64);
  * `Generator.random` = (next_uint64 >> 11) * 2**-53;
  * `Generator.integers`, `Generator.permutation` (host-side scalars/permutations);
  * stable `np.lexsort`, `np.unique`.
`oracle/pcg64.py` restates the PCG64 arithmetic so the GPU replay can be
checked draw-by-draw.
"""
