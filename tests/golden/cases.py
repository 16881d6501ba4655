"""Regenerable inputs of the golden training cases (no reference import, so the
GPU box can rebuild them).  Used by make_golden.py and the tests."""

import numpy as np

from oracle import tfhe32 as o
from paper_2403_20190_b200.params import named_params

TRAIN_CASES = {
    # name: (params name, p, (s, l, a, r), samples, key seed, enc seed, data seed)
    "train_cfg1": ("CFG1", 16, (120, 2, 4, 7), 3, 4, 5, 6),      # z = 0: rotation only
    "train_tree": ("CFG2", 256, (50, 10, 12, 7), 2, 4, 5, 6),     # z = 6 tree + clear padding bits
}


def train_inputs(name):
    """(params, s1, bits, labels, per-sample RGSW stacks) of a training case,
    encrypted by the oracle at q = 2^32 (hw/hewnn.py:109-119 stream order)."""
    pname, p, (s, l, a, r), count, kseed, eseed, dseed = TRAIN_CASES[name]
    P = named_params(pname, p)
    s1 = o.make_rng(kseed).integers(0, 2, P.n).astype(np.uint32)
    drng = np.random.default_rng(dseed)
    bits = drng.integers(0, 2, (count, s))
    labels = drng.integers(0, l, count)
    lb = max(1, (l - 1).bit_length())
    rng = o.make_rng(eseed)
    g = P.gadget
    stacks = []
    for i in range(count):
        data = o.enc_rgsw_batch(bits[i], s1, P.sigma, g.levels, g.base_log, rng)
        lab = o.enc_rgsw_batch([(labels[i] >> b) & 1 for b in range(lb)], s1, P.sigma, g.levels, g.base_log, rng)
        stacks.append(np.concatenate([data, lab]))
    return P, s1, bits, labels, stacks
