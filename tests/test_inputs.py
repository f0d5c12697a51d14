"""The seeded input generator (shared by oracle and product; holds no method arithmetic)."""
import numpy as np

import hkinputs as gen

MASK = (1 << 64) - 1


def _splitmix_py(c):
    z = ((c + 1) * 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def test_splitmix_matches_scalar_reference():
    w = gen.raw_words(7, 1, 5, 9)
    for e in range(5):
        for k in range(9):
            c = (((7 * 4 + 1) << 32) + e) << 12 | k
            assert int(w[e, k]) == _splitmix_py(c & MASK)


def test_known_splitmix_value():
    # SplitMix64 with state 0: first output is 0xe220a8397b1dcdaf (widely published)
    assert _splitmix_py(0) == 0xE220A8397B1DCDAF
    assert int(gen.splitmix64(np.zeros(1, dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_uniform_layout_and_canonical_form():
    for P in (1, 63, 64, 65, 3328, 33216):
        m, s = gen.uniform(3, 0, 50, P)
        L = gen.n_limbs(P)
        assert m.shape == (50, L) and m.dtype == np.uint64 and s.dtype == np.int8
        assert np.all(m[:, L - 1] & ~gen.top_mask(P) == 0)
        assert np.all((s == 0) == (~m.any(axis=1)))
        assert set(np.unique(s)).issubset({-1, 0, 1})


def test_deterministic_and_streams_differ():
    a1 = gen.uniform(2, 0, 10, 500)[0]
    a2 = gen.uniform(2, 0, 10, 500)[0]
    x1 = gen.uniform(2, 1, 10, 500)[0]
    assert np.array_equal(a1, a2) and not np.array_equal(a1, x1)


def test_carry_stress_structure():
    P = 16608
    m, s = gen.carry_stress(4, 0, 40, P)
    full = gen.max_magnitude(1, P)[0][0]
    for e in range(0, 40, 2):
        assert np.array_equal(m[e], full)
        assert s[e] == (1 if (e // 2) % 2 == 0 else -1)
    odd = m[1::2]
    assert (~odd.any(axis=1)).sum() > 0 and odd.any(axis=1).sum() > 0


def test_config_shapes():
    for name, c in gen.CONFIGS.items():
        if c["n"] > 1024:
            continue
        am, asg, xm, xsg = gen.config_inputs(name)
        assert am.shape[0] == gen.a_count(c["kind"], c["n"]) and xm.shape[0] == c["n"]
