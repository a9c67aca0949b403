"""CPU-only tests: C-ABI surface, host-side mirror logic, validation, sharding plumbing."""

import ctypes as C
import math
import os
import re

import numpy as np
import pytest
import torch

import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import _lib
from conftest import ROOT, load_golden


def header_symbols():
    text = open(os.path.join(ROOT, "include", "svgear.h")).read()
    return sorted(set(re.findall(r"\b(svgear_[a-z_0-9]+)\s*\(", text)))


class TestCAbi:
    def test_library_loads_and_exports_every_declared_symbol(self):
        handle = C.CDLL(_lib.build_library())
        names = header_symbols()
        assert len(names) >= 11
        for n in names:
            assert hasattr(handle, n), n
        assert set(names) == set(_lib.SIGNATURES), "ctypes table out of sync with include/svgear.h"

    def test_version_and_strerror(self):
        lib = P.load_library()
        assert lib.svgear_version() == 111
        assert lib.svgear_strerror(0) == b"ok"
        assert b"workspace" in lib.svgear_strerror(_lib.EWORKSPACE)

    def test_workspace_query_and_shape_rejection(self):
        n = _lib.workspace_bytes(_lib.Shape(2, 4096, 4096, 64, 32, 64))
        assert 0 < n < (1 << 32)
        for bad in (_lib.Shape(1, 16, 16, 32, 2, 2), _lib.Shape(1, 16, 16, 64, 17, 2),
                    _lib.Shape(0, 16, 16, 64, 2, 2), _lib.Shape(1, 16, 16, 64, 2, 0)):
            out = C.c_size_t(0)
            assert P.load_library().svgear_workspace_bytes(C.byref(bad), C.byref(out)) == _lib.ESHAPE

    def test_argument_errors_precede_device_errors(self):
        lib = P.load_library()
        # null pointers -> EINVAL, bad iteration count -> EINVAL, bad d -> ESHAPE
        assert lib.svgear_kmeans(0, 1, 8, 64, 2, None, None, 5, None, None, None, None, None, None, None,
                                 None, 0, None) == _lib.EINVAL
        buf = (C.c_char * 4096)()
        p = C.addressof(buf)
        assert lib.svgear_kmeans(0, 1, 8, 64, 2, p, p, 0, p, p, p, p, p, None, None, p, 4096, None) == _lib.EINVAL
        assert lib.svgear_kmeans(0, 1, 8, 48, 2, p, p, 5, p, p, p, p, p, None, None, p, 4096, None) == _lib.ESHAPE
        assert lib.svgear_route_error_aware(1, 1, 2, p, p, p, -1, 0, 1, p, None, p, 4096, None) == _lib.EINVAL

    @pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
    def test_compute_entries_fail_loudly_without_a_device(self):
        lib = P.load_library()
        buf = (C.c_char * 4096)()
        p = C.addressof(buf)
        assert lib.svgear_kmeans(0, 1, 8, 64, 2, p, p, 5, p, p, p, p, p, None, None, p, 4096, None) == _lib.ECUDA
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            P.svg_ear_attention(*(torch.zeros(8, 64, dtype=torch.bfloat16),) * 3, 2, 2, 0.25)


class TestHeadGroupLayout:
    """Host-side plan of the operator's head groups (operator._group_layout): groups partition the
    instances contiguously and the workspace of a split call is the aligned sum of its groups'."""

    def test_partition_and_workspace(self):
        from paper_2603_08982_b200 import operator as op
        for bh, groups in ((40, 2), (40, 3), (5, 5), (7, 4), (24, 1)):
            bnd, needs, total = op._group_layout(bh, 4096, 4096, 64, 32, 64, groups)
            assert bnd[0] == 0 and bnd[-1] == bh and len(bnd) == groups + 1
            sizes = [b - a for a, b in zip(bnd, bnd[1:])]
            assert all(s >= 1 for s in sizes) and max(sizes) - min(sizes) <= 1
            for s, n in zip(sizes, needs):
                assert n >= _lib.workspace_bytes(_lib.Shape(s, 4096, 4096, 64, 32, 64))
                assert groups == 1 or n % 256 == 0
            assert total == sum(needs) + (256 if groups > 1 else 0)

    def test_operator_workspace_bytes(self):
        one = P.operator_workspace_bytes(40, 75600, 75600, 128, 300, 1000, head_groups=1)
        assert one == _lib.workspace_bytes(_lib.Shape(40, 75600, 75600, 128, 300, 1000))
        auto = P.operator_workspace_bytes(40, 75600, 75600, 128, 300, 1000)
        two = P.operator_workspace_bytes(40, 75600, 75600, 128, 300, 1000, head_groups=2)
        assert auto == two  # >= 16 large instances -> two groups
        assert abs(two - one) < 0.01 * one  # splitting costs alignment, not memory
        assert P.operator_workspace_bytes(8, 75600, 75600, 128, 300, 1000) == \
            _lib.workspace_bytes(_lib.Shape(8, 75600, 75600, 128, 300, 1000))
        assert P.operator_workspace_bytes(3, 512, 512, 64, 4, 4, head_groups=9) == \
            P.operator_workspace_bytes(3, 512, 512, 64, 4, 4, head_groups=3)

    def test_seeded_forward_argument_errors(self):
        lib = P.load_library()
        buf = (C.c_char * 4096)()
        p = C.addressof(buf)
        shape = _lib.Shape(1, 256, 256, 64, 8, 8)
        tail = (5, 0, 100, 0, 1, 0, 0.0, p, p, None, p, 4096, None)
        fwd = lambda oversample, first, sh=shape: lib.svgear_forward_seeded(C.byref(sh), p, p, p, oversample, 0, first,
                                                                            p, p, *tail)
        assert fwd(0, 0) == _lib.EINVAL     # no subsample
        assert fwd(9, 0) == _lib.EINVAL     # beyond what the workspace is sized for
        assert fwd(8, -1) == _lib.EINVAL    # negative instance index
        assert lib.svgear_forward_seeded(None, p, p, p, 8, 0, 0, p, p, *tail) == _lib.EINVAL
        bad = _lib.Shape(1, 256, 256, 96, 8, 8)
        assert fwd(8, 0, bad) == _lib.ESHAPE
        # standalone seeding: argument checks come before any device work
        assert lib.svgear_kmeans_seed(1, 256, 64, 8, None, 8, 0, 0, p, p, 4096, None) == _lib.EINVAL
        assert lib.svgear_kmeans_seed(1, 256, 64, 8, p, 0, 0, 0, p, p, 4096, None) == _lib.EINVAL
        assert lib.svgear_kmeans_seed(1, 256, 64, 300, p, 8, 0, 0, p, p, 4096, None) == _lib.ESHAPE


class TestValidationMirrorsReference:
    def test_budget(self):  # tests/test_router.py:52-73
        assert P.DensityBudget.global_density(0.25).rho == 0.25
        assert P.DensityBudget.top_p(0.85).p == 0.85
        for rho in (-0.1, 1.1, None):
            with pytest.raises(ValueError, match="rho"):
                P.DensityBudget(mode="globalDensity", rho=rho)
        for p in (0.0, -0.5, 1.5, None):
            with pytest.raises(ValueError, match="p"):
                P.DensityBudget(mode="perClusterTopP", p=p)
        with pytest.raises(ValueError, match="mode"):
            P.DensityBudget(mode="entryBudget", rho=0.5)
        with pytest.raises(ValueError, match="overshoot"):
            P.DensityBudget(mode="globalDensity", rho=0.5, overshoot="panic")

    def test_entry_capacity(self):  # tests/test_router.py:76-85
        assert P.entry_capacity(0.25, 65536) == 16384
        assert P.entry_capacity(0.7, 10) == 7 and P.entry_capacity(0.3, 10) == 3
        assert P.entry_capacity(0.25, 75600 * 75600) == 1428840000  # needs 64-bit

    def test_kmeans_argument_errors(self):  # clustering.py:166-175, linalg.py:28-31
        x = np.zeros((8, 64), dtype=np.float32)
        with pytest.raises(ValueError, match=">= 1"):
            P.kmeans(x, 0)
        with pytest.raises(ValueError, match="exceeds"):
            P.kmeans(x, 9)
        with pytest.raises(ValueError, match="restarts"):
            P.kmeans(x, 2, restarts=0)
        with pytest.raises(ValueError, match="max_iters"):
            P.kmeans(x, 2, max_iters=0)
        with pytest.raises(P.ShapeError):
            P.kmeans(np.zeros((2, 2, 2, 64)), 1)
        bad = x.copy()
        bad[0, 0] = np.nan
        with pytest.raises(ValueError, match="non-finite"):
            P.kmeans(bad, 2)

    def test_operator_argument_errors(self):
        t = torch.zeros(1, 2, 16, 64, dtype=torch.bfloat16)
        with pytest.raises(ValueError, match="rho"):
            P.svg_ear_attention(t, t, t, 2, 2, 1.5)
        with pytest.raises(ValueError, match="exceeds"):
            P.svg_ear_attention(t, t, t, 17, 2, 0.5)
        with pytest.raises(ValueError, match="estimator"):
            P.svg_ear_attention(t, t, t, 2, 2, 0.5, estimator="fancy")
        with pytest.raises(ValueError, match="differ"):
            P.svg_ear_attention(t, t, t[:, :, :8], 2, 2, 0.5)
        with pytest.raises(P.ShapeError):
            P.svg_ear_attention(t[..., :32], t[..., :32], t[..., :32], 2, 2, 0.5)
        with pytest.raises(ValueError, match="estimator"):
            P.build_error_table(None, "bogus")

    def test_seed_recipe_matches_reference_golden(self):
        # the product-side k-means++ start must be the reference's (clustering.py:65-84,178-180)
        g = load_golden("pipeline_gauss_d64")
        qs, ks = P.analysis.side_seeds(int(g["seed"]))
        q = g["q"].astype(np.float64)
        k = g["k"].astype(np.float64)
        assert np.array_equal(P.clustering.seeded_start(q, int(g["c_q"]), qs), g["q_init"])
        assert np.array_equal(P.clustering.seeded_start(k, int(g["c_k"]), ks), g["k_init"])

    def test_flop_closed_forms(self):  # attention.py:212-219
        assert P.exact_block_flops(64, 1000) == 256000
        assert P.compensation_flops(8, [2, 3], [1, 4]) == 4 * 8 * 14


class TestShardingPlan:
    def test_head_ranges_partition_exactly(self):
        for heads, world in ((40, 1), (40, 2), (40, 8), (24, 8), (24, 5), (3, 8)):
            spans = [P.head_range(heads, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == heads
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
        assert P.head_range(40, 8, 3) == (15, 20)
        with pytest.raises(ValueError):
            P.head_range(4, 2, 2)
