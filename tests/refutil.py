"""Helpers that run the Python reference (``/root/reference``) -- build container only.

The reference does not exist on the GPU box; tests that need it skip there.  GPU tests use
the committed golden fixtures (``tests/golden``) and the C oracle instead.
"""
from __future__ import annotations

import os
import sys

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HAVE_REF = os.path.isdir(REF_SRC)

if HAVE_REF:
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)


def ref():
    """The reference package ``lsd_wfst`` (raises ImportError off the build container)."""
    import lsd_wfst  # noqa: F401
    import lsd_wfst.decoder
    import lsd_wfst.fixtures
    import lsd_wfst.lattice
    import lsd_wfst.parallel
    import lsd_wfst.posteriors
    import lsd_wfst.wfst
    return lsd_wfst


def ref_oracles():
    """The reference's brute-force path enumerators (pkg/tests/oracles.py)."""
    if REF_TESTS not in sys.path:
        sys.path.insert(0, REF_TESTS)
    import oracles  # noqa: F401
    return oracles


def ref_cost_table(posts):
    """Cost table built row by row with the reference's own ``frame_costs``."""
    import numpy as np
    from lsd_wfst.posteriors import frame_costs
    T, L1 = posts.rows.shape
    out = np.empty((T, L1), dtype=np.float64)
    for f in range(T):
        out[f] = frame_costs(posts, f, 1.0)
    return out


def random_instance(seed, *, max_states=12, max_arcs=30, max_frames=6, num_labels=3,
                    eps_fraction=0.15, blank_fraction=0.0, weight_grid=None, selfloops=False):
    """Same envelope as the reference's tests/conftest.py:52-66."""
    import random
    L = ref()
    rng = random.Random(seed)
    states = rng.randrange(2, max_states + 1)
    arcs = rng.randrange(states, max_arcs + 1)
    frames = rng.randrange(0, max_frames + 1)
    labels = rng.randrange(1, num_labels + 1)
    wfst = L.fixtures.make_random_wfst(rng, states, arcs, labels, eps_fraction=eps_fraction,
                                       selfloops=selfloops, weight_grid=weight_grid)
    posts = L.fixtures.make_random_posteriors(rng, frames, labels, blank_fraction=blank_fraction)
    return wfst, posts


def oracle_instance(seed):
    """Criterion-1 envelope of the reference acceptance suite (test_acceptance.py:65-83)."""
    import random
    L = ref()
    rng = random.Random(seed)
    states = rng.randrange(2, 13)
    arcs = rng.randrange(states, 31)
    labels = rng.randrange(1, 5)
    selfloops = seed % 4 == 0
    frames = rng.randrange(0, 5 if selfloops else 7)
    wfst = L.fixtures.make_random_wfst(rng, states, arcs, labels,
                                       eps_fraction=0.1 if seed % 3 == 0 else 0.0,
                                       selfloops=selfloops, final_fraction=0.5)
    posts = L.fixtures.make_random_posteriors(rng, frames, labels,
                                              blank_fraction=0.3 if seed % 2 else 0.0)
    return wfst, posts


def equivalence_instance(seed):
    """Criterion-5 envelope (test_acceptance.py:235-273): returns (wfst, posts, cfg kwargs)."""
    import math
    import random
    L = ref()
    INF = math.inf
    rng = random.Random(seed)
    bucket = seed % 20
    if bucket == 19:
        states = rng.randrange(100, 201); arcs = rng.randrange(2 * states, 3 * states)
        frames = rng.randrange(12, 21); grid = None; eps = 0.1
    elif bucket == 9:
        states = rng.randrange(40, 81); arcs = rng.randrange(states, 2 * states)
        frames = rng.randrange(6, 13); grid = None; eps = 0.15
    elif bucket in (4, 14):
        states = rng.randrange(6, 25); arcs = rng.randrange(2 * states, 4 * states)
        frames = rng.randrange(2, 7); grid = [0.0, 0.5, 1.0]; eps = 0.2
    else:
        states = rng.randrange(3, 31); arcs = rng.randrange(states, 3 * states)
        frames = rng.randrange(1, 7); grid = None; eps = 0.15 if seed % 3 == 0 else 0.0
    labels = rng.randrange(2, 5)
    wfst = L.fixtures.make_random_wfst(rng, states, arcs, labels, eps_fraction=eps,
                                       selfloops=bucket % 2 == 0, weight_grid=grid)
    posts = L.fixtures.make_random_posteriors(rng, frames, labels,
                                              blank_fraction=0.3 if seed % 2 else 0.0)
    cfg = dict(mode="lsd" if seed % 2 else "fsd", beam=(INF, 6.0, 3.0)[seed % 3],
               max_active=(None, 8, 24)[seed % 3])
    return wfst, posts, cfg
