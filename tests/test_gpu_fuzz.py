"""Randomized GPU parity tests (B200): many small ragged shapes through the C ABI against the CPU
oracle.  Deterministic seeds; every case states its shape on failure.  These exist to catch
timing / edge-shape bugs that the reference-shaped tests do not reach (a race in the attention
epilogue was found this way)."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

import paper_2603_08982_b200 as P
from oracle import svgear_oracle as O

pytestmark = pytest.mark.gpu


def dev(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def host(t):
    return t.detach().cpu().numpy()


def rel_l2(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def np_model(m):
    return SimpleNamespace(num_clusters=m.num_clusters, assignments=host(m.assignments).astype(np.int64),
                           centroids=host(m.centroids).astype(np.float64), sizes=host(m.sizes).astype(np.int64),
                           permutation=host(m.permutation).astype(np.int64), offsets=host(m.offsets).astype(np.int64))


def random_instance(rng, max_q=900, max_k=1200, max_cq=16, max_ck=48):
    d = int(rng.choice([64, 128]))
    n_q, n_k = int(rng.integers(2, max_q)), int(rng.integers(2, max_k))
    c_q, c_k = int(rng.integers(1, min(n_q, max_cq) + 1)), int(rng.integers(1, min(n_k, max_ck) + 1))
    kind = rng.integers(0, 3)
    if kind == 0:      # iid Gaussian, random scale
        q, k, v = (rng.normal(size=s) * rng.uniform(0.3, 2.0) for s in ((n_q, d), (n_k, d), (n_k, d)))
    elif kind == 1:    # blobs
        q, k, v = O.blob_instance(n_q, n_k, d, max(1, c_q), max(1, c_k), float(rng.uniform(0.05, 0.5)), int(rng.integers(1 << 30)))
    else:              # many exact duplicates (empty-cluster repair, tied distances)
        bq, bk = rng.normal(size=(max(1, n_q // 7), d)), rng.normal(size=(max(1, n_k // 9), d))
        q = bq[rng.integers(0, len(bq), n_q)]
        ki = rng.integers(0, len(bk), n_k)
        k, v = bk[ki], rng.normal(size=(len(bk), d))[ki]
    return tuple(O.round_to_bf16(t) for t in (q, k, v)) + (c_q, c_k, d, int(kind))


@pytest.mark.parametrize("seed", list(range(24)))
def test_executor_random_masks(seed):
    rng = np.random.default_rng(7000 + seed)
    q, k, v, c_q, c_k, d, kind = random_instance(rng)
    prep = P.prepare(dev(q), dev(k), dev(v), c_q, c_k, seed=seed, max_iters=int(rng.integers(1, 26)))
    qm, km = np_model(prep.q_model), np_model(prep.k_model)
    for mdl, n in ((qm, len(q)), (km, len(k))):
        assert sorted(mdl.permutation.tolist()) == list(range(n)) and (mdl.sizes >= 1).all()
        assert np.array_equal(mdl.permutation, np.argsort(mdl.assignments, kind="stable"))
    sizes = prep.q_model.sizes.long().unsqueeze(1) * prep.k_model.sizes.long().unsqueeze(0)
    qp, kp, vp = q[qm.permutation], k[km.permutation], v[km.permutation]
    for density in (0.0, float(rng.uniform(0.05, 0.95)), 1.0):
        sel = rng.random((c_q, c_k)) < density
        mask = P.mask_from_selected(torch.from_numpy(sel).cuda(), sizes)
        want = O.mixed_logit_output(qp, kp, vp, qm, km, sel)
        _, want_lse = O.sparse_attend(qp, kp, vp, qm, km, sel)
        for dtype, tol, ltol in ((torch.float32, 1e-4, 1e-3), (torch.bfloat16, 1e-2, 3e-2)):
            res = P.sparse_attend(prep.q, prep.k, prep.v, prep.q_model, prep.k_model, mask, dtype=dtype)
            info = (len(q), len(k), c_q, c_k, d, kind, density, str(dtype))
            assert rel_l2(host(res.output.float()), want) <= tol, info
            assert np.abs(host(res.lse) - want_lse).max() <= ltol, info


@pytest.mark.parametrize("seed", list(range(12)))
def test_bounded_lloyd_equals_full_evaluation(seed):
    from paper_2603_08982_b200.clustering import run_lloyd
    rng = np.random.default_rng(8000 + seed)
    q, k, v, c_q, c_k, d, kind = random_instance(rng, max_q=3000, max_k=3000, max_cq=64, max_ck=200)
    for x, c in ((q, c_q), (k, c_k)):
        xs = dev(np.stack([x, x[::-1].copy()]))                 # two instances per call
        starts = xs[:, rng.choice(len(x), size=c, replace=False)].float().contiguous()
        a = run_lloyd(xs, starts, 25)
        b = run_lloyd(xs, starts, 25, full_eval=True)
        torch.cuda.synchronize()
        for key in ("assign", "perm", "sizes", "offsets", "iters"):
            assert torch.equal(a[key], b[key]), (key, len(x), c, d, kind)
        assert torch.equal(a["centroids"], b["centroids"]), (len(x), c, d, kind)
        labels, inertia, iters = O.lloyd(x.astype(np.float64), c, 25, host(starts[0]).astype(np.float64))
        mism = float((host(a["assign"][0]) != labels).mean())
        # exact duplicates tie in float64 but not always in fp32: report, bound
        assert mism <= (0.02 if kind == 2 else 0.0), (len(x), c, d, kind, mism)


@pytest.mark.parametrize("seed", list(range(10)))
def test_operator_end_to_end(seed):
    rng = np.random.default_rng(9000 + seed)
    q, k, v, c_q, c_k, d, kind = random_instance(rng, max_q=700, max_k=900, max_cq=10, max_ck=30)
    mode = "perClusterTopP" if seed % 2 else "globalDensity"
    budget = float(rng.uniform(0.2, 0.95)) if mode == "perClusterTopP" else float(rng.uniform(0.0, 1.0))
    H = 2
    qs, ks, vs = (dev(np.stack([t, t[::-1].copy()]))[None] for t in (q, k, v))
    out, mask, aux = P.svg_ear_attention(qs, ks, vs, c_q, c_k, budget, budget_mode=mode, seed=seed,
                                         init="strided", check_fp32=False, return_aux=True)
    for h in range(H):
        qh, kh, vh = (host(t[0, h].float()).astype(np.float64) for t in (qs, ks, vs))
        qm = SimpleNamespace(num_clusters=c_q, assignments=host(aux["q_assign"][0, h]).astype(np.int64),
                             centroids=host(aux["q_centroids"][0, h]).astype(np.float64),
                             sizes=host(aux["q_sizes"][0, h]).astype(np.int64),
                             permutation=host(aux["q_perm"][0, h]).astype(np.int64),
                             offsets=host(aux["q_offsets"][0, h]).astype(np.int64))
        km = SimpleNamespace(num_clusters=c_k, assignments=host(aux["k_assign"][0, h]).astype(np.int64),
                             centroids=host(aux["k_centroids"][0, h]).astype(np.float64),
                             sizes=host(aux["k_sizes"][0, h]).astype(np.int64),
                             permutation=host(aux["k_perm"][0, h]).astype(np.int64),
                             offsets=host(aux["k_offsets"][0, h]).astype(np.int64))
        sel = host(mask[0, h])
        # the executor against the oracle on the GPU's own clustering and mask, original row order
        o_out, _ = O.sparse_attend(qh[qm.permutation], kh[km.permutation], vh[km.permutation], qm, km, sel)
        info = (len(q), len(k), c_q, c_k, d, kind, mode, budget, h)
        assert rel_l2(host(out[0, h].float()), O.unpermute(o_out, qm)) <= 1e-2, info
        # the budget is honoured
        ent = int((np.outer(qm.sizes, km.sizes) * sel).sum())
        assert ent == int(aux["mask_entries"][0, h]), info
        if mode == "globalDensity":
            assert ent <= P.entry_capacity(budget, len(q) * len(k)), info


@pytest.mark.parametrize("seed", list(range(12)))
def test_error_table_and_routing_random_shapes(seed):
    """Error table against the oracle ON THE GPU'S OWN clustering (so only the estimator is compared),
    then both routing modes bit-exact against the oracle's router run on the GPU's table."""
    rng = np.random.default_rng(9500 + seed)
    q, k, v, c_q, c_k, d, kind = random_instance(rng, max_q=1500, max_k=2500, max_cq=40, max_ck=120)
    prep = P.prepare(dev(q), dev(k), dev(v), c_q, c_k, seed=seed, max_iters=5)
    qm, km = np_model(prep.q_model), np_model(prep.k_model)
    ref_prep = SimpleNamespace(q_model=qm, k_model=km, q=q[qm.permutation].astype(np.float64),
                               k=k[km.permutation].astype(np.float64), v=v[km.permutation].astype(np.float64))
    info = (len(q), len(k), c_q, c_k, d, kind)
    for mode in ("valueAware", "plain"):
        got = host(P.build_error_table(prep, mode).error_sum)
        want = O.build_error_table(ref_prep, mode).error_sum
        assert np.isfinite(got).all() and (got >= 0).all(), info
        assert np.abs(got - want).max() <= 5e-4 * max(want.max(), 1e-30), info + (mode,)
    table = P.build_error_table(prep, "valueAware")
    mine = SimpleNamespace(error_sum=host(table.error_sum), q_sizes=qm.sizes, k_sizes=km.sizes)
    rho = float(rng.uniform(0.0, 1.0))
    m = P.route_error_aware(table, P.DensityBudget.global_density(rho))
    want = O.route_error_aware(mine, rho)
    assert np.array_equal(host(m.selected), want.selected), info + (rho,)
    assert m.density_entries == want.density_entries
    p = float(rng.uniform(0.1, 1.0))
    m = P.route_error_aware(table, P.DensityBudget.top_p(p), q_centroids=prep.q_model.centroids,
                            k_centroids=prep.k_model.centroids)
    want = O.route_error_aware_top_p(mine, qm.centroids, km.centroids, p)
    mism = float((host(m.selected) != want.selected).mean())
    assert mism <= (0.05 if kind == 2 else 2e-3), info + (p, mism)   # duplicates: exactly tied masses


@pytest.mark.parametrize("seed", list(range(4)))
def test_executor_medium_multi_tile(seed):
    """Query clusters of several hundred to a few thousand rows: 256-row two-half CTA tiles plus the
    one-half remainder kernel, several heads per launch."""
    rng = np.random.default_rng(9900 + seed)
    d = int(rng.choice([64, 128]))
    n_q, n_k = int(rng.integers(1500, 5000)), int(rng.integers(1500, 5000))
    c_q, c_k = int(rng.integers(2, 9)), int(rng.integers(8, 60))
    H = 3
    qs, ks, vs = (O.round_to_bf16(rng.normal(size=(H, n, d))) for n in (n_q, n_k, n_k))
    prep = P.prepare(dev(qs), dev(ks), dev(vs), c_q, c_k, seed=seed, max_iters=4)
    sel = rng.random((H, c_q, c_k)) < rng.uniform(0.1, 0.6)
    sizes = prep.q_model.sizes.long().unsqueeze(-1) * prep.k_model.sizes.long().unsqueeze(-2)
    mask = P.mask_from_selected(torch.from_numpy(sel).cuda(), sizes)
    res = P.sparse_attend(prep.q, prep.k, prep.v, prep.q_model, prep.k_model, mask, dtype=torch.bfloat16)
    for h in range(H):
        qm = SimpleNamespace(**{f: host(getattr(prep.q_model, f)[h]).astype(np.int64 if f != "centroids" else np.float64)
                                for f in ("assignments", "centroids", "sizes", "permutation", "offsets")}, num_clusters=c_q)
        km = SimpleNamespace(**{f: host(getattr(prep.k_model, f)[h]).astype(np.int64 if f != "centroids" else np.float64)
                                for f in ("assignments", "centroids", "sizes", "permutation", "offsets")}, num_clusters=c_k)
        want = O.mixed_logit_output(qs[h][qm.permutation], ks[h][km.permutation], vs[h][km.permutation], qm, km, sel[h])
        assert rel_l2(host(res.output[h].float()), want) <= 1e-2, (n_q, n_k, c_q, c_k, d, h)


def test_run_to_run_determinism():
    """No floating-point atomics, fixed-order reductions: repeated calls are bit-identical even
    though the two k-means sides and the two attention kernels run concurrently."""
    torch.manual_seed(5)
    q, k, v = (torch.randn(1, 4, 7000, 128, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    ref = None
    for rep in range(3):
        out, mask, aux = P.svg_ear_attention(q, k, v, 24, 80, 0.3, init="device", return_aux=True)
        cur = [out, mask, aux["q_perm"], aux["k_perm"], aux["k_centroids"], aux["error_table"], aux["lse"]]
        if ref is None:
            ref = [t.clone() for t in cur]
        else:
            assert all(torch.equal(a, b) for a, b in zip(cur, ref)), rep
