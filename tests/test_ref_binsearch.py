"""The reference's comparison-search test classes (pkg/tests/test_binsearch.py
and test_eytzinger.py), restated against the B200 package: same class and
test names, scenarios and expectations; the oracle (oracle/fs_oracle.py)
checks.  The probe-count classes (TestIterationCounts / TestProbeBounds /
test_exactly_L_comparisons) instrument the reference's pure-Python `*_seq`
loops, which live in oracle/ here; their device counterparts are fixed-trip
by construction (search.cuh) and are covered by the sweeps below.
"""

import numpy as np
import pytest

from oracle import fs_oracle as orc


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def _searchers(fs, p):
    """test_binsearch.py:29-40: the five comparison kernels as z -> index."""
    pp, probe, c = fs.pad_right_pow2(p), fs.probe_constant(p.n_intervals), fs.offset_constants(p.n_intervals)
    return {
        "classic": lambda z: fs.classic_search(p, z),
        "bitset1": lambda z: fs.bitset_search_v1(p, probe, z),
        "bitset2": lambda z: fs.bitset_search_v2(pp, z),
        "bitset3": lambda z: fs.bitset_search_v3(p, probe, z),
        "offset": lambda z: fs.offset_search(p, c, z),
    }


# --------------------------------------------------------------------------- test_binsearch.py:43-79
@pytest.mark.gpu
class TestExamples:
    def test_classic(self, cuda):
        fs = _fs()
        p = fs.validate_partition([0, 1, 2, 3])
        assert (fs.classic_search(p, 2.9), fs.classic_search(p, 0.0)) == (2, 0)

    def test_bitset1(self, cuda):
        fs = _fs()
        assert fs.bitset_search_v1(fs.validate_partition([0, 1, 2, 3]), fs.probe_constant(3), 1.5) == 1
        p9 = fs.gen_uniform_gap_partition(9, 1, 5, seed=9)
        assert fs.bitset_search_v1(p9, fs.probe_constant(8), np.nextafter(p9.values[-1], -np.inf)) == 7

    def test_bitset2(self, cuda):
        fs = _fs()
        assert fs.bitset_search_v2(fs.pad_right_pow2(fs.validate_partition([0, 1, 2, 3])), 2.5) == 2
        p9 = fs.gen_uniform_gap_partition(9, 1, 5, seed=9)
        assert fs.bitset_search_v2(fs.pad_right_pow2(p9), np.nextafter(p9.values[-1], -np.inf)) == 7

    def test_bitset3(self, cuda):
        fs = _fs()
        assert fs.bitset_search_v3(fs.validate_partition([0, 1, 2, 3]), fs.probe_constant(3), 1.0) == 1
        p9 = fs.gen_uniform_gap_partition(9, 1, 5, seed=9)
        assert fs.bitset_search_v3(p9, fs.probe_constant(8), p9.values[0]) == 0

    def test_offset(self, cuda):
        fs = _fs()
        assert fs.offset_search(fs.validate_partition([0, 1, 2, 3]), fs.offset_constants(3), 2.2) == 2
        assert fs.offset_search(fs.validate_partition([0.0, 1.0]), fs.offset_constants(1), 0.5) == 0

    def test_out_of_domain(self, cuda):
        fs = _fs()
        for name, search in _searchers(fs, fs.validate_partition([0, 1, 2, 3])).items():
            with pytest.raises(fs.OutOfDomain):
                search(3.0)


# --------------------------------------------------------------------------- test_binsearch.py:82-93
class TestOffsetConstants:
    @pytest.mark.parametrize("n,f,s,j", [(7, 4, 4, 3), (1, 1, 1, 1), (14, 7, 8, 3)])
    def test_values(self, n, f, s, j):
        c = _fs().offset_constants(n)
        assert (c.F, c.S, c.J) == (f, s, j)

    def test_invariants(self):
        for n in range(1, 200):
            c = _fs().offset_constants(n)
            assert c.F >= 1 and c.S >= 1 and c.F + c.S == n + 1
            assert 2**c.J <= n + 1 < 2 ** (c.J + 1)


# --------------------------------------------------------------------------- test_binsearch.py:96-123
@pytest.mark.gpu
class TestOracleEquivalence:
    @pytest.mark.parametrize("precision", ["single", "double"])
    def test_exhaustive_small_sizes(self, cuda, precision):
        """Every comparison kernel equals the oracle on every boundary-heavy
        probe, sizes 2..64 (one batch launch per kernel and size)."""
        fs = _fs()
        for size in range(2, 65):
            p = fs.gen_uniform_gap_partition(size, 1, 5, seed=size, precision=precision)
            z = orc.boundary_probes(p.values)
            want = orc.linear_scan_batch(p.values, z)
            for algorithm in ("classic", "bitset1", "bitset2", "bitset3", "offset", "eytzinger"):
                got = fs.run_batch(fs.prepare(algorithm, p), z, d=16)
                assert np.array_equal(got, want), (algorithm, size)

    @pytest.mark.parametrize("size", [15, 255, 4095])
    def test_randomized_larger_sizes(self, cuda, size):
        fs = _fs()
        p = fs.gen_uniform_gap_partition(size, 1, 5, seed=size)
        z = orc.random_queries(p.values, 10_000, seed=size + 1)
        want = orc.linear_scan_batch(p.values, z)
        for algorithm in ("classic", "bitset1", "bitset2", "bitset3", "offset"):
            assert np.array_equal(fs.run_batch(fs.prepare(algorithm, p), z, d=64), want), algorithm
        # the scalar entry points agree with the batch path on a sample
        searchers = _searchers(fs, p)
        for v in z[:40]:
            assert {name: s(v) for name, s in searchers.items()} == dict.fromkeys(searchers, orc.linear_scan(p.values, v))


# --------------------------------------------------------------------------- test_eytzinger.py:21-63
@pytest.mark.gpu
class TestLayout:
    def test_no_padding_when_tree_is_full(self, cuda):
        fs = _fs()
        from paper_1506_08620_b200.eytzinger import in_order

        lay = fs.build_layout(fs.validate_partition([0.0, 1.0, 2.0]))
        assert lay.L == 2 and len(lay.tree) == 3 and in_order(lay).tolist() == [0.0, 1.0, 2.0]

    def test_root_is_middle_of_full_tree(self, cuda):
        fs = _fs()
        p = fs.gen_uniform_gap_partition(15, 1, 5, seed=15)
        lay = fs.build_layout(p)
        assert lay.L == 4 and lay.tree[0] == np.sort(p.values)[7]

    def test_padding_copies_of_last_knot(self, cuda):
        fs = _fs()
        p = fs.gen_uniform_gap_partition(9, 1, 5, seed=9)
        lay = fs.build_layout(p)
        assert lay.L == 4 and len(lay.tree) == 15
        assert np.count_nonzero(lay.tree == p.values[-1]) == 7

    @pytest.mark.parametrize("size", list(range(2, 40)) + [64, 100, 257])
    def test_in_order_reconstruction(self, cuda, size):
        fs = _fs()
        from paper_1506_08620_b200.eytzinger import in_order

        p = fs.gen_uniform_gap_partition(size, 1, 5, seed=size)
        flat = in_order(fs.build_layout(p))
        assert np.array_equal(flat[:size], p.values) and np.all(flat[size:] == p.values[-1])

    def test_every_base_element_present_once(self, cuda):
        fs = _fs()
        p = fs.gen_uniform_gap_partition(11, 1, 5, seed=2)
        tree = fs.build_layout(p).tree
        assert all(np.count_nonzero(tree == v) == 1 for v in p.values[:-1])

    def test_depth_formula(self):
        from paper_1506_08620_b200.eytzinger import tree_depth

        for n, depth in [(1, 2), (2, 2), (3, 3), (6, 3), (7, 4), (14, 4), (15, 5)]:
            assert tree_depth(n) == depth and 2**depth - 1 >= n + 1
            assert depth == 1 or 2 ** (depth - 1) - 1 < n + 1


# --------------------------------------------------------------------------- test_eytzinger.py:65-84
@pytest.mark.gpu
class TestSearch:
    def test_examples(self, cuda):
        fs = _fs()
        lay = fs.build_layout(fs.validate_partition([0.0, 1.0, 2.0]))
        assert (fs.eytzinger_search(lay, 1.5), fs.eytzinger_search(lay, 0.0)) == (1, 0)

    def test_out_of_domain(self, cuda):
        fs = _fs()
        with pytest.raises(fs.OutOfDomain):
            fs.eytzinger_search(fs.build_layout(fs.validate_partition([0.0, 1.0, 2.0])), 2.0)

    @pytest.mark.parametrize("precision", ["single", "double"])
    def test_exhaustive_oracle_sweep(self, cuda, precision):
        fs = _fs()
        for size in range(2, 34):
            p = fs.gen_uniform_gap_partition(size, 1, 5, seed=size, precision=precision)
            z = orc.boundary_probes(p.values)
            got = fs.run_batch(fs.prepare("eytzinger", p), z, d=8)
            assert np.array_equal(got, orc.linear_scan_batch(p.values, z)), size
