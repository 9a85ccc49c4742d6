"""ORACLE (test infrastructure): K^π values of single CSR node rows, for sampled
parity at sizes where the full oracle pattern is too large (cfg5: 2.9e9 nnz).
Same scatter rule as assemble.scatter (reading R9)."""
from __future__ import annotations

import numpy as np

from .dofmap import row_contributions


def row_block_values(prob, dm, pairs, local_of, I, locs=None):
    """(cols J, blocks (nb, d, d)) of node row I; local_of(t) -> (n_rows_tile, d, d)."""
    d = prob.d
    cols, contribs = row_contributions(prob, dm, pairs, I, locs)
    out = np.zeros((len(cols), d, d))
    cache = {}
    for n, lst in enumerate(contribs):
        for t, r, tr in lst:
            if t not in cache:
                cache[t] = local_of(t)
            L = cache[t][r]
            if cols[n] == I:                      # diagonal block: symmetric upper entry
                out[n] += np.triu(L) + np.triu(L, 1).T
            elif tr:
                out[n] += L.T
            else:
                out[n] += L
    return np.array(cols), out
