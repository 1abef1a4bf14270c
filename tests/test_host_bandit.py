"""Host-side pieces of the device bandit: the numpy-backed reveal trace and the PCG64 seeding shortcut."""

import numpy as np
import pytest

from paper_2602_02827_b200.bandit import Reveals, RunResult, _rng_state, pcg64_seed_state


def test_reveals_behave_like_the_reference_list():
    ref = [(3, 1, 0.25), (0, 4, -0.5), (3, 0, 1.0)]
    r = Reveals(np.array([3, 0, 3]), np.array([1, 4, 0]), np.array([0.25, -0.5, 1.0]))
    assert r == ref and ref == r and not (r != ref)
    assert r == [list(x) for x in ref]  # golden JSON holds lists
    assert r != ref[:2] and r != [(3, 1, 0.25), (0, 4, -0.5), (3, 0, 1.5)]
    assert len(r) == 3 and r[1] == (0, 4, -0.5) and r[-1] == (3, 0, 1.0) and r[:2] == ref[:2]
    assert list(r) == ref and [tuple(x) for x in r] == ref
    i, t, v = r[0]
    assert type(i) is int and type(t) is int and type(v) is float
    assert r == Reveals.from_list(ref) and Reveals.from_list([]) == []
    assert RunResult([3], 0.5, r, 2, "separation") == RunResult([3], 0.5, ref, 2, "separation")


@pytest.mark.parametrize("seed", [0, 1, 7, 2 ** 32 + 5, 2 ** 70, (0, 0), (0, 255), (4, 1, 9), [2, 3]])
def test_pcg64_seed_state_equals_numpy(seed):
    st = np.random.default_rng(seed).bit_generator.state
    assert pcg64_seed_state(seed) == (st["state"]["state"], st["state"]["inc"])
    p, warm = _rng_state(seed, "epsilon-greedy", 0.0, 100)
    assert (p.state_hi << 64 | p.state_lo) == st["state"]["state"]
    assert (p.inc_hi << 64 | p.inc_lo) == st["state"]["inc"] and p.has_uint32 == 0 and len(warm) == 0


def test_static_warmup_state_follows_the_choice_draw():
    g = np.random.default_rng((0, 3))
    cells = g.choice(60, size=6, replace=False)
    st = g.bit_generator.state
    p, warm = _rng_state((0, 3), "static-warmup", 0.1, 60)
    assert warm.tolist() == cells.tolist()
    assert (p.state_hi << 64 | p.state_lo) == st["state"]["state"]
    assert p.has_uint32 == st["has_uint32"] and p.uinteger == st["uinteger"]


def test_numpy_descriptor_view_matches_the_ctypes_struct():
    """prepare_batch fills cbx_bandit_run_desc column-wise through a numpy view: same bytes as ctypes."""
    from paper_2602_02827_b200 import _lib
    from paper_2602_02827_b200.bandit import _desc_dtype

    dt = _desc_dtype()
    assert dt.itemsize == 152
    d = _lib.CbxBanditRunDesc()
    a = np.zeros(1, dtype=dt)
    vals = dict(query=7, row_begin=123456789012, n_rows=1000, n_cols=100, k=10, explore_mode=2, n_warm=5, flags=3,
                warm_off=99, alpha_ef=0.178, epsilon=0.1, log_term=12.5, bounds_off=-1, lo_uniform=-1.0,
                hi_uniform=1.0, trace_off=2 ** 40, state_off=2 ** 33)
    for k, v in vals.items():
        setattr(d, k, v)
        a[k] = v
    rng = (2 ** 63 + 5, 17, 2 ** 64 - 1, 3, 1, 2 ** 32 - 2)
    d.rng = _lib.CbxPcg64(*rng)
    for sub, v in zip(("state_hi", "state_lo", "inc_hi", "inc_lo", "has_uint32", "uinteger"), rng):
        a["rng_" + sub] = v
    assert a.tobytes() == bytes(d)
