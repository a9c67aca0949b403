"""Generate tests/golden/*.npz by running the REAL reference package.

Run in the build container only (the reference is mounted read-only at
/root/reference and does not exist on the GPU box):

    python oracle/make_golden.py

Every array stored here is an output of `routedattn` itself (not of the
restatement in oracle/svgear_oracle.py), so the fixtures pin both the oracle
(tests/test_oracle_pinned.py, CPU) and the CUDA path (tests/test_gpu_*.py).
Inputs are rounded to bf16-representable values first so the float64 reference
and the bf16 GPU operator consume identical numbers.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import routedattn  # noqa: E402  (the reference)
from routedattn import analysis, attention, clustering, estimator, router  # noqa: E402
from routedattn.oracle import full_attention  # noqa: E402

from oracle.svgear_oracle import round_to_bf16  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
RHOS = (0.0, 0.1, 0.25, 0.5, 1.0)


def _inputs(kind, n_q, n_k, d, c_q, c_k, seed):
    if kind == "blobs":
        q, k, v = analysis.make_blob_instance(
            analysis.BlobSpec(n_q, n_k, d, q_blobs=c_q, k_blobs=c_k, sigma=0.1), seed)
    elif kind == "gauss":
        rng = np.random.default_rng(seed)
        q, k, v = rng.normal(size=(n_q, d)), rng.normal(size=(n_k, d)), rng.normal(size=(n_k, d))
    elif kind == "dups":
        q, k, v, _, _ = analysis.make_duplicate_instance(n_q, n_k, d, c_q, c_k, seed)
    else:
        raise ValueError(kind)
    return round_to_bf16(q), round_to_bf16(k), round_to_bf16(v)


def pipeline_case(name, kind, n_q, n_k, d, c_q, c_k, seed):
    q, k, v = _inputs(kind, n_q, n_k, d, c_q, c_k, seed)
    q_seed, k_seed = (int(s) for s in np.random.SeedSequence(seed).generate_state(2))
    q_init = clustering._kmeans_pp_init(
        q, c_q, np.random.default_rng(np.random.SeedSequence(entropy=q_seed, spawn_key=(0,))))
    k_init = clustering._kmeans_pp_init(
        k, c_k, np.random.default_rng(np.random.SeedSequence(entropy=k_seed, spawn_key=(0,))))
    prep = analysis.prepare(q, k, v, c_q, c_k, seed=seed)
    qm, km = prep.q_model, prep.k_model
    t_stream = analysis.build_error_table(prep, "valueAware")
    t_naive = estimator.estimate_errors_value_aware(qm, km, prep.k, prep.v)
    t_plain = analysis.build_error_table(prep, "plain")
    rec = dict(
        q=q.astype(np.float32), k=k.astype(np.float32), v=v.astype(np.float32),
        c_q=c_q, c_k=c_k, seed=seed, q_init=q_init, k_init=k_init,
        q_assign=qm.assignments, k_assign=km.assignments,
        q_perm=qm.permutation, k_perm=km.permutation,
        q_sizes=qm.sizes, k_sizes=km.sizes, q_offsets=qm.offsets, k_offsets=km.offsets,
        q_centroids=qm.centroids, k_centroids=km.centroids,
        v_centroids=clustering.segment_means(prep.v, km),
        err_stream=t_stream.error_sum, err_naive=t_naive.error_sum, err_plain=t_plain.error_sum,
        stabilizers=t_stream.stabilizers,
        rank_order=np.array([b.q_cluster * c_k + b.k_cluster for b in estimator.to_ratios(t_stream)]),
        rhos=np.array(RHOS), dense=full_attention(q, k, v)[1],
    )
    for r in RHOS:
        tag = f"{int(round(r * 100)):03d}"
        m = router.route_error_aware(t_stream, router.DensityBudget.global_density(r))
        m_stop = router.route_error_aware(
            t_stream, router.DensityBudget.global_density(r, router.STOP_AT_FIRST_OVERFLOW))
        m_nofb = router.route_error_aware(t_stream, router.DensityBudget.global_density(r),
                                          single_item_fallback=False)
        m_score = router.route_score(qm.centroids, km.centroids, qm.sizes, km.sizes,
                                     router.DensityBudget.global_density(r))
        res = attention.sparse_attend(prep.q, prep.k, prep.v, qm, km, m)
        rec[f"mask_{tag}"] = m.selected
        rec[f"mask_stop_{tag}"] = m_stop.selected
        rec[f"mask_nofb_{tag}"] = m_nofb.selected
        rec[f"mask_score_{tag}"] = m_score.selected
        rec[f"entries_{tag}"] = m.density_entries
        rec[f"out_perm_{tag}"] = res.output
        rec[f"lse_perm_{tag}"] = res.lse
        rec[f"out_{tag}"] = clustering.inverse_permute_rows(res.output, qm)
        rec[f"flops_exact_{tag}"] = res.flops.exact_block
        rec[f"flops_comp_{tag}"] = res.flops.compensation
    for p in (0.5, 0.85, 1.0):
        tag = f"{int(round(p * 100)):03d}"
        rec[f"mask_topp_{tag}"] = router.route_error_aware(
            t_stream, router.DensityBudget.top_p(p),
            q_centroids=qm.centroids, k_centroids=km.centroids).selected
        rec[f"mask_scoretopp_{tag}"] = router.score_top_p(
            qm.centroids, km.centroids, qm.sizes, km.sizes, p).selected
    np.savez_compressed(os.path.join(OUT, f"pipeline_{name}.npz"), **rec)
    print(f"pipeline_{name}: iters unknown, sizes q={qm.sizes.min()}..{qm.sizes.max()} "
          f"k={km.sizes.min()}..{km.sizes.max()} density@.25={rec['entries_025'] / (n_q * n_k):.4f}")


def router_tables():
    """Random small tables -> reference masks, to pin the greedy walk, the
    fallback and both overshoot policies independent of clustering."""
    rng = np.random.default_rng(2024)
    recs = {}
    n = 0
    for trial in range(24):
        cq, ck = int(rng.integers(1, 6)), int(rng.integers(1, 9))
        qs = rng.integers(1, 12, size=cq)
        ks = rng.integers(1, 20, size=ck)
        err = rng.random((cq, ck)) ** 3 * np.outer(qs, ks)
        if trial % 5 == 0:  # exact ratio ties and zeros
            err = np.round(err)
        table = estimator.BlockErrorTable(error_sum=err, q_sizes=qs, k_sizes=ks,
                                          stabilizers=np.zeros(cq), mode="valueAware", flops=0)
        for cap_frac in (0.0, 0.07, 0.3, 0.6, 1.0):
            cap = int(cap_frac * int(qs.sum()) * int(ks.sum()))
            for ov in (router.FILL_REMAINDER, router.STOP_AT_FIRST_OVERFLOW):
                for fb in (True, False):
                    m = router.route_error_aware_entries(table, cap, overshoot=ov,
                                                         single_item_fallback=fb)
                    recs[f"err_{n}"] = err
                    recs[f"qs_{n}"] = qs
                    recs[f"ks_{n}"] = ks
                    recs[f"cap_{n}"] = cap
                    recs[f"stop_{n}"] = ov == router.STOP_AT_FIRST_OVERFLOW
                    recs[f"fb_{n}"] = fb
                    recs[f"sel_{n}"] = m.selected
                    n += 1
    recs["count"] = n
    np.savez_compressed(os.path.join(OUT, "router_tables.npz"), **recs)
    print("router_tables:", n, "cases")


def kmeans_cases():
    """k-means from explicit warm starts (init_centroids) and from seeds, incl.
    the duplicate-token repair case of tests/test_clustering.py:88-94."""
    recs = {}
    rng = np.random.default_rng(77)
    # duplicates: only 3 distinct rows but k=5 forces the empty-cluster repair
    base = round_to_bf16(rng.normal(size=(3, 64)))
    x = np.repeat(base, 8, axis=0)[rng.permutation(24)]
    m = clustering.kmeans(x, 5, seed=3)
    init = clustering._kmeans_pp_init(
        x, 5, np.random.default_rng(np.random.SeedSequence(entropy=3, spawn_key=(0,))))
    recs.update(dup_x=x.astype(np.float32), dup_init=init, dup_assign=m.assignments,
                dup_perm=m.permutation, dup_sizes=m.sizes, dup_centroids=m.centroids)
    # SPEC.md:123 example
    x1 = np.array([[0.0], [0.0], [10.0], [10.0]])
    m1 = clustering.kmeans(x1, 2, seed=0)
    recs.update(spec_assign=m1.assignments, spec_centroids=m1.centroids)
    np.savez_compressed(os.path.join(OUT, "kmeans_cases.npz"), **recs)
    print("kmeans_cases: dup sizes", m.sizes)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    print("reference version", routedattn.__version__)
    pipeline_case("blobs_d64", "blobs", 256, 320, 64, 8, 12, seed=0)
    pipeline_case("gauss_d64", "gauss", 192, 224, 64, 6, 9, seed=1)
    pipeline_case("gauss_d128", "gauss", 160, 160, 128, 5, 7, seed=2)
    pipeline_case("dups_d64", "dups", 128, 128, 64, 4, 8, seed=3)
    pipeline_case("tiny_d16", "gauss", 40, 48, 16, 3, 4, seed=5)
    router_tables()
    kmeans_cases()
