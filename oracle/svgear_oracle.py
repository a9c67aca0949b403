"""CPU oracle for the SVG-EAR attention hot path (TEST INFRASTRUCTURE ONLY).

This file is a float64 numpy restatement of the algorithm the reference
package `routedattn` (mounted read-only at /root/reference/pkg/src/routedattn)
runs for the path

    prepare -> build_error_table -> route_error_aware -> sparse_attend

It is NOT part of the product: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it, and only
as the checker / the CPU arm.  The CUDA operator never calls into this module
and has no CPU fallback.

Pinning: `tests/test_oracle_pinned.py` checks every function here against the
golden vectors the reference's own tests hold for the path (router known-answer
vectors, entry_capacity vectors, ranking tie rules, executor identities) and
against fixtures under `tests/golden/` that were produced by importing the real
reference in the build container (`oracle/make_golden.py`).  All integer / index
outputs (assignments, permutations, masks) are compared bit-exactly, floats to
<= 1e-12.

Every function cites the reference lines it restates as  [ref: file:line].
Arithmetic is kept in the same operation order as the reference wherever the
order is observable (distance expansion, argmin tie rule, sequential row
accumulation of cluster means, streaming rescale, greedy walk).
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

F64 = np.float64


# ----------------------------------------------------------------------------
# input validation                                   [ref: linalg.py:21-32]
# ----------------------------------------------------------------------------
def token_matrix(x):
    a = np.ascontiguousarray(x, dtype=F64)
    if a.ndim != 2:
        raise ValueError(f"token matrix must be 2-D, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("token matrix contains non-finite entries")
    return a


# ----------------------------------------------------------------------------
# clustering                                         [ref: clustering.py]
# ----------------------------------------------------------------------------
def side_seeds(seed):
    """(q_seed, k_seed) derivation used by prepare.   [ref: analysis.py:227]"""
    s = np.random.SeedSequence(seed).generate_state(2)
    return int(s[0]), int(s[1])


def restart_rng(side_seed, restart=0):
    """Generator for one k-means restart.            [ref: clustering.py:178-180]"""
    return np.random.default_rng(np.random.SeedSequence(entropy=side_seed, spawn_key=(restart,)))


def squared_distances(x, c):
    """|x|^2 - 2 x.c + |c|^2 clipped at zero.         [ref: clustering.py:55-62]"""
    xx = (x * x).sum(axis=1, keepdims=True)
    cc = (c * c).sum(axis=1)
    return np.maximum(xx - 2.0 * (x @ c.T) + cc, 0.0)


def kmeanspp_centres(x, k, rng):
    """k-means++ seeding with the reference's RNG call sequence.
    [ref: clustering.py:65-84]"""
    n, d = x.shape
    out = np.empty((k, d), dtype=x.dtype)
    used = np.zeros(n, dtype=bool)
    pick = int(rng.integers(n))
    out[0] = x[pick]
    used[pick] = True
    near = ((x - out[0]) ** 2).sum(axis=1)
    for j in range(1, k):
        tot = near.sum()
        if tot > 0.0:
            pick = int(rng.choice(n, p=near / tot))
        else:
            pick = int(np.flatnonzero(~used)[0])
        out[j] = x[pick]
        used[pick] = True
        near = np.minimum(near, ((x - out[j]) ** 2).sum(axis=1))
    return out


def pad_centres(x, centres, k):
    """Warm-start padding by farthest token.          [ref: clustering.py:87-101]"""
    centres = np.array(centres, dtype=F64, copy=True)
    if centres.ndim != 2 or centres.shape[1] != x.shape[1]:
        raise ValueError(
            f"init centroids must be 2-D with {x.shape[1]} columns, got {centres.shape}")
    if centres.shape[0] > k:
        raise ValueError(f"got {centres.shape[0]} init centroids for {k} clusters")
    near = squared_distances(x, centres).min(axis=1)
    while centres.shape[0] < k:
        far = int(np.argmax(near))
        centres = np.vstack([centres, x[far]])
        near = np.minimum(near, ((x - x[far]) ** 2).sum(axis=1))
    return centres


def member_mean(x, idx):
    """Mean of gathered member rows (ascending order). [ref: clustering.py:49-52]"""
    return x[idx].mean(axis=0)


def means_by_label(x, labels, k):
    return np.stack([member_mean(x, np.flatnonzero(labels == c)) for c in range(k)])


def lloyd(x, k, max_iters, centres):
    """Lloyd iterations with lowest-index ties and empty-cluster repair.
    Returns (labels, inertia, iterations).            [ref: clustering.py:104-141]"""
    n = x.shape[0]
    last = None
    last_inertia = np.inf
    labels = np.zeros(n, dtype=np.int64)
    iters = 0
    for _ in range(max_iters):
        iters += 1
        dist = squared_distances(x, centres)
        labels = dist.argmin(axis=1)
        own = dist[np.arange(n), labels]
        counts = np.bincount(labels, minlength=k)
        for c in np.flatnonzero(counts == 0):
            can_give = np.flatnonzero(counts[labels] >= 2)
            giver = can_give[np.argmax(own[can_give])]
            counts[labels[giver]] -= 1
            counts[c] += 1
            labels[giver] = c
            centres = centres.copy()
            centres[c] = x[giver]
            own[giver] = 0.0
        inertia = float(own.sum())
        last_inertia = inertia
        if last is not None and np.array_equal(labels, last):
            break
        last = labels
        centres = means_by_label(x, labels, k)
    return labels, last_inertia, iters


def cluster_model(x, labels, k, iters=0):
    """Final model from labels.                       [ref: clustering.py:193-207]"""
    sizes = np.bincount(labels, minlength=k)
    return SimpleNamespace(
        num_clusters=k,
        assignments=labels,
        centroids=means_by_label(x, labels, k),
        sizes=sizes,
        permutation=np.argsort(labels, kind="stable"),
        offsets=np.concatenate(([0], np.cumsum(sizes)[:-1])),
        iters=iters,
    )


def kmeans(x, k, *, max_iters=25, seed=0, restarts=1, init_centroids=None, starts=None):
    """[ref: clustering.py:144-207].  `starts` (list of explicit start centre
    sets) is an oracle-only convenience used to feed the GPU and the oracle the
    identical initialisation."""
    x = token_matrix(x)
    n = x.shape[0]
    if k < 1:
        raise ValueError(f"num_clusters must be >= 1, got {k}")
    if k > n:
        raise ValueError(f"num_clusters ({k}) exceeds token count ({n})")
    if restarts < 1:
        raise ValueError(f"restarts must be >= 1, got {restarts}")
    if max_iters < 1:
        raise ValueError(f"max_iters must be >= 1, got {max_iters}")
    if starts is None:
        starts = [kmeanspp_centres(x, k, restart_rng(seed, r)) for r in range(restarts)]
        if init_centroids is not None:
            starts.append(pad_centres(x, init_centroids, k))
    best = None
    for c0 in starts:
        labels, inertia, iters = lloyd(x, k, max_iters, np.asarray(c0, dtype=F64))
        if best is None or inertia < best[1]:
            best = (labels, inertia, iters)
    return cluster_model(x, best[0], k, best[2])


def segment_means(xp, model):
    """Per-cluster means of a cluster-contiguous matrix. [ref: clustering.py:247-257]"""
    out = np.empty((model.num_clusters, xp.shape[1]), dtype=xp.dtype)
    for c in range(model.num_clusters):
        a = int(model.offsets[c])
        out[c] = xp[a:a + int(model.sizes[c])].mean(axis=0)
    return out


def prepare(q, k, v, c_q, c_k, *, seed=0, q_starts=None, k_starts=None, max_iters=25):
    """Cluster both sides, permute cluster-contiguous. [ref: analysis.py:207-239]"""
    q = token_matrix(q)
    k = token_matrix(k)
    v = token_matrix(v)
    if k.shape[0] != v.shape[0]:
        raise ValueError(f"key/value row counts differ: {k.shape[0]} vs {v.shape[0]}")
    qs, ks = side_seeds(seed)
    qm = kmeans(q, c_q, seed=qs, max_iters=max_iters, starts=q_starts)
    km = kmeans(k, c_k, seed=ks, max_iters=max_iters, starts=k_starts)
    return SimpleNamespace(q_raw=q, k_raw=k, v_raw=v, q_model=qm, k_model=km,
                           q=q[qm.permutation], k=k[km.permutation], v=v[km.permutation])


def reference_init_centres(q, k, c_q, c_k, seed):
    """The k-means++ centres `prepare(seed=...)` starts from (restart 0), so the
    GPU path can be handed the identical initialisation.
    [ref: analysis.py:227 + clustering.py:178-180 + clustering.py:65-84]"""
    qs, ks = side_seeds(seed)
    return (kmeanspp_centres(token_matrix(q), c_q, restart_rng(qs)),
            kmeanspp_centres(token_matrix(k), c_k, restart_rng(ks)))


# ----------------------------------------------------------------------------
# error estimation                                   [ref: estimator.py]
# ----------------------------------------------------------------------------
def _table(err, qm, km, stab, mode):
    return SimpleNamespace(error_sum=err, q_sizes=qm.sizes.copy(), k_sizes=km.sizes.copy(),
                           stabilizers=stab, mode=mode)


def error_table_streaming(qm, km, kp, vp, *, tile=64):
    """Value-aware block errors, streamed in key tiles with running-max rescale;
    accumulator starts at zero.                        [ref: estimator.py:187-253]"""
    if tile < 1:
        raise ValueError(f"tile_size must be >= 1, got {tile}")
    d = kp.shape[1]
    scale = 1.0 / math.sqrt(d)
    qbar = qm.centroids.astype(F64)
    kbar = km.centroids.astype(F64)
    vbar = segment_means(vp, km).astype(F64)
    sbar = (qbar @ kbar.T) * F64(scale)
    m_ref = sbar.max(axis=1)
    cq = qm.num_clusters
    err = np.empty((cq, km.num_clusters), dtype=F64)
    for j in range(km.num_clusters):
        a = int(km.offsets[j])
        b = a + int(km.sizes[j])
        m_loc = m_ref.copy()
        wbar = np.exp(sbar[:, j] - m_loc)
        acc = np.zeros(cq, dtype=F64)
        for t0 in range(a, b, tile):
            t1 = min(t0 + tile, b)
            logits = (qbar @ kp[t0:t1].T) * F64(scale)
            m_new = np.maximum(m_loc, logits.max(axis=1))
            alpha = np.exp(m_loc - m_new)
            acc *= alpha * alpha
            wbar *= alpha
            e = np.exp(logits - m_new[:, None])
            r = wbar[:, None, None] * vbar[j][None, None, :] - e[:, :, None] * vp[t0:t1][None, :, :]
            acc += (r * r).sum(axis=(1, 2))
            m_loc = m_new
        err[:, j] = acc * np.exp(2.0 * (m_loc - m_ref))
    err = qm.sizes[:, None] * err
    return _table(np.asarray(err, dtype=F64), qm, km, np.asarray(m_ref, dtype=F64), "valueAware")


def error_table_value_aware(qm, km, kp, vp):
    """Direct Eq.8 table.                              [ref: estimator.py:151-184]"""
    d = kp.shape[1]
    sbar = (qm.centroids @ km.centroids.T) / math.sqrt(d)
    c = sbar.max(axis=1)
    vbar = segment_means(vp, km)
    logits = (qm.centroids @ kp.T) / math.sqrt(d)
    ebar = np.repeat(np.exp(sbar - c[:, None]), km.sizes, axis=1)
    ekey = np.exp(logits - c[:, None])
    vrows = np.repeat(vbar, km.sizes, axis=0)
    r = ebar[:, :, None] * vrows[None, :, :] - ekey[:, :, None] * vp[None, :, :]
    per_key = (r * r).sum(axis=2)
    err = qm.sizes[:, None] * np.add.reduceat(per_key, km.offsets, axis=1)
    return _table(err, qm, km, c, "valueAware")


def error_table_plain(qm, km, kp):
    """Plain Eq.5 table.                               [ref: estimator.py:120-148]"""
    d = kp.shape[1]
    sbar = (qm.centroids @ km.centroids.T) / math.sqrt(d)
    c = sbar.max(axis=1)
    logits = (qm.centroids @ kp.T) / math.sqrt(d)
    ebar = np.exp(sbar - c[:, None])
    ekey = np.exp(logits - c[:, None])
    diff = np.repeat(ebar, km.sizes, axis=1) - ekey
    err = qm.sizes[:, None] * np.add.reduceat(diff * diff, km.offsets, axis=1)
    return _table(err, qm, km, c, "plain")


def build_error_table(prep, mode="valueAware", tile=64):
    """[ref: analysis.py:242-249]"""
    if mode == "valueAware":
        return error_table_streaming(prep.q_model, prep.k_model, prep.k, prep.v, tile=tile)
    if mode == "plain":
        return error_table_plain(prep.q_model, prep.k_model, prep.k)
    raise ValueError(f"unknown estimator mode {mode!r}")


# ----------------------------------------------------------------------------
# routing                                            [ref: router.py, estimator.py:83-96]
# ----------------------------------------------------------------------------
FILL_REMAINDER = "fillRemainder"
STOP_AT_FIRST_OVERFLOW = "stopAtFirstOverflow"


def block_sizes(table):
    return np.outer(table.q_sizes, table.k_sizes)


def ranked_order(table):
    """Flat block indices in the total order (-ratio, -error, qc, kc).
    [ref: estimator.py:83-96].  lexsort on the same float64 keys gives the same
    order as the reference's Python tuple sort."""
    w = block_sizes(table).reshape(-1)
    e = table.error_sum.reshape(-1)
    ratio = e / w
    flat = np.arange(e.size)
    return flat[np.lexsort((flat, -e, -ratio))]


def entry_capacity(rho, total):
    """[ref: router.py:93-97]"""
    return int(math.floor(rho * total + 1e-9))


def greedy_walk(order, weights, capacity, overshoot=FILL_REMAINDER):
    """[ref: router.py:100-110]"""
    take = []
    left = int(capacity)
    for i in order:
        w = int(weights[i])
        if w <= left:
            take.append(int(i))
            left -= w
        elif overshoot == STOP_AT_FIRST_OVERFLOW:
            break
    return take


def single_block_rescue(take, values, weights, capacity):
    """[ref: router.py:113-121]"""
    fits = np.flatnonzero(weights <= capacity)
    if fits.size == 0:
        return take
    best = fits[np.argmax(values[fits])]
    if values[best] > sum(float(values[i]) for i in take):
        return [int(best)]
    return take


def _mask(selected, sizes):
    """[ref: router.py:81-85]"""
    selected = np.asarray(selected, dtype=bool)
    ent = int(sizes[selected].sum())
    return SimpleNamespace(selected=selected, density_entries=ent, density=ent / int(sizes.sum()))


def route_error_aware_entries(table, capacity, *, overshoot=FILL_REMAINDER, fallback=True):
    """[ref: router.py:124-142]"""
    cq, ck = table.error_sum.shape
    sizes = block_sizes(table)
    w = sizes.reshape(-1)
    val = table.error_sum.reshape(-1)
    take = greedy_walk(ranked_order(table), w, capacity, overshoot)
    if fallback:
        take = single_block_rescue(take, val, w, capacity)
    sel = np.zeros(cq * ck, dtype=bool)
    sel[take] = True
    return _mask(sel.reshape(cq, ck), sizes)


def route_error_aware(table, rho, *, overshoot=FILL_REMAINDER, fallback=True):
    """globalDensity mode.                             [ref: router.py:145-171]"""
    if not (0.0 <= rho <= 1.0):
        raise ValueError(f"globalDensity budget needs rho in [0, 1], got {rho}")
    total = int(table.q_sizes.sum()) * int(table.k_sizes.sum())
    return route_error_aware_entries(table, entry_capacity(rho, total),
                                     overshoot=overshoot, fallback=fallback)


def softmax_rows(a):
    """[ref: linalg.py:49-61]"""
    w = np.exp(a - a.max(axis=1, keepdims=True))
    return w / w.sum(axis=1, keepdims=True)


def cluster_scores(qc, kc, k_sizes, size_weighted=True):
    """[ref: router.py:193-206]"""
    s = (qc @ kc.T) / math.sqrt(qc.shape[1])
    if size_weighted:
        s = s + np.log(k_sizes.astype(F64))
    return s


def score_top_p(qc, kc, q_sizes, k_sizes, p, *, size_weighted=True):
    """[ref: router.py:209-236]"""
    if not (0.0 < p <= 1.0):
        raise ValueError(f"p must be in (0, 1], got {p}")
    mass = softmax_rows(cluster_scores(qc, kc, k_sizes, size_weighted))
    cq, ck = mass.shape
    sel = np.zeros((cq, ck), dtype=bool)
    for i in range(cq):
        if p == 1.0:
            sel[i] = True
            continue
        order = np.argsort(-mass[i], kind="stable")
        cut = int(np.searchsorted(np.cumsum(mass[i][order]), p, side="left"))
        sel[i, order[: min(cut, ck - 1) + 1]] = True
    return _mask(sel, np.outer(q_sizes, k_sizes))


def route_error_aware_top_p(table, qc, kc, p, *, overshoot=FILL_REMAINDER, fallback=True,
                            size_weighted=True):
    """perClusterTopP mode.                            [ref: router.py:172-190, 239-250]"""
    cq, ck = table.error_sum.shape
    sizes = block_sizes(table)
    caps = (score_top_p(qc, kc, table.q_sizes, table.k_sizes, p,
                        size_weighted=size_weighted).selected * sizes).sum(axis=1).astype(np.int64)
    order = ranked_order(table)
    sel = np.zeros((cq, ck), dtype=bool)
    for i in range(cq):
        row = [int(b % ck) for b in order if b // ck == i]
        take = greedy_walk(row, sizes[i], int(caps[i]), overshoot)
        if fallback:
            take = single_block_rescue(take, table.error_sum[i], sizes[i], int(caps[i]))
        sel[i, take] = True
    return _mask(sel, sizes)


def route_score(qc, kc, q_sizes, k_sizes, rho, *, overshoot=FILL_REMAINDER, size_weighted=True):
    """SVG2-style mass routing at a global density.    [ref: router.py:253-280]"""
    mass = softmax_rows(cluster_scores(qc, kc, k_sizes, size_weighted))
    sizes = np.outer(q_sizes, k_sizes)
    cq, ck = mass.shape
    fm = mass.reshape(-1)
    flat = np.arange(fm.size)
    order = flat[np.lexsort((flat, -fm))]
    take = greedy_walk(order, sizes.reshape(-1), entry_capacity(rho, int(sizes.sum())), overshoot)
    sel = np.zeros(cq * ck, dtype=bool)
    sel[take] = True
    return _mask(sel.reshape(cq, ck), sizes)


# ----------------------------------------------------------------------------
# executor                                           [ref: attention.py]
# ----------------------------------------------------------------------------
def exact_pass(qp, kp, vp, qm, km, selected, dtype=F64):
    """[ref: attention.py:57-101]"""
    qp = qp.astype(dtype, copy=False)
    kp = kp.astype(dtype, copy=False)
    vp = vp.astype(dtype, copy=False)
    scale = 1.0 / math.sqrt(qp.shape[1])
    out = np.zeros((qp.shape[0], vp.shape[1]), dtype=dtype)
    lse = np.full(qp.shape[0], -np.inf, dtype=dtype)
    entries = 0
    for i in range(qm.num_clusters):
        a = int(qm.offsets[i])
        rows = slice(a, a + int(qm.sizes[i]))
        picked = np.flatnonzero(selected[i])
        if picked.size == 0:
            continue
        cols = np.concatenate([np.arange(int(km.offsets[j]), int(km.offsets[j]) + int(km.sizes[j]))
                               for j in picked])
        s = (qp[rows] @ kp[cols].T) * scale
        m = s.max(axis=1)
        w = np.exp(s - m[:, None])
        z = w.sum(axis=1)
        out[rows] = (w @ vp[cols]) / z[:, None]
        lse[rows] = m + np.log(z)
        entries += int(qm.sizes[i]) * cols.size
    return out, lse, entries


def compensate(qp, km, vbar, qm, selected, part_out, part_lse, dtype=F64):
    """[ref: attention.py:104-157]"""
    if selected.shape[1] == 0:
        raise ValueError("no key clusters: softmax over an empty set is undefined")
    qp = qp.astype(dtype, copy=False)
    kbar = km.centroids.astype(dtype, copy=False)
    vbar = vbar.astype(dtype, copy=False)
    scale = 1.0 / math.sqrt(qp.shape[1])
    lnw = np.log(km.sizes.astype(F64)).astype(dtype)
    out = np.array(part_out, copy=True)
    lse = np.array(part_lse, copy=True)
    for i in range(qm.num_clusters):
        todo = [j for j in range(km.num_clusters) if not selected[i, j]]
        if not todo:
            continue
        a = int(qm.offsets[i])
        rows = slice(a, a + int(qm.sizes[i]))
        m = lse[rows].copy()
        l = np.ones(int(qm.sizes[i]), dtype=dtype)
        acc = out[rows].copy()
        for j in todo:
            s = (qp[rows] @ kbar[j]) * scale + lnw[j]
            m_new = np.maximum(m, s)
            alpha = np.exp(m - m_new)
            p = np.exp(s - m_new)
            l = l * alpha + p
            acc = acc * alpha[:, None] + p[:, None] * vbar[j]
            m = m_new
        out[rows] = acc / l[:, None]
        lse[rows] = m + np.log(l)
    return out, lse


def sparse_attend(qp, kp, vp, qm, km, selected, dtype=F64):
    """[ref: attention.py:160-192].  Returns (output, lse) in permuted row order."""
    with np.errstate(invalid="ignore"):
        po, pl, _ = exact_pass(qp, kp, vp, qm, km, selected, dtype)
        return compensate(qp, km, segment_means(vp, km), qm, selected, po, pl, dtype)


def mixed_logit_output(qp, kp, vp, qm, km, selected):
    """Dense Eq.1 reference.        [ref: attention.py:195-209, oracle.py:59-78]"""
    d = qp.shape[1]
    krows = np.repeat(km.centroids, km.sizes, axis=0)
    entry = np.repeat(np.repeat(selected, qm.sizes, axis=0), km.sizes, axis=1)
    logits = np.where(entry, (qp @ kp.T) / math.sqrt(d), (qp @ krows.T) / math.sqrt(d))
    probs = softmax_rows(logits)
    vrows = np.repeat(segment_means(vp, km), km.sizes, axis=0)
    return (probs * entry) @ vp + (probs * ~entry) @ vrows


def dense_attention(q, k, v):
    """[ref: oracle.py:52-56]"""
    return softmax_rows((q @ k.T) / math.sqrt(q.shape[1])) @ v


def unpermute(rows, model):
    """[ref: clustering.py:215-219]"""
    out = np.empty_like(rows)
    out[model.permutation] = rows
    return out


# ----------------------------------------------------------------------------
# the operator: four-call composition     [ref: cli.py:119-134, README.md:94-98]
# ----------------------------------------------------------------------------
def forward(q, k, v, c_q, c_k, rho, *, seed=0, q_starts=None, k_starts=None, max_iters=25,
            estimator="valueAware", overshoot=FILL_REMAINDER, fallback=True):
    """One (Q,K,V) head through the whole path.  Output is returned both in the
    reference's permuted row order and in original token order."""
    prep = prepare(q, k, v, c_q, c_k, seed=seed, q_starts=q_starts, k_starts=k_starts,
                   max_iters=max_iters)
    table = build_error_table(prep, estimator)
    mask = route_error_aware(table, rho, overshoot=overshoot, fallback=fallback)
    out_p, lse_p = sparse_attend(prep.q, prep.k, prep.v, prep.q_model, prep.k_model, mask.selected)
    return SimpleNamespace(prep=prep, table=table, mask=mask, out_permuted=out_p, lse_permuted=lse_p,
                           out=unpermute(out_p, prep.q_model), lse=unpermute(lse_p, prep.q_model))


# closed-form work model                [ref: attention.py:212-219, estimator.py:42-47,
#                                             clustering.py:138-140]
def flops_exact(d, entries):
    return 4 * d * int(entries)


def flops_compensation(d, q_sizes, n_comp_per_row):
    return int(4 * d * (np.asarray(q_sizes) * np.asarray(n_comp_per_row)).sum())


def flops_estimation(d, c_q, n_k):
    return c_q * n_k * (6 * d + 4)


def flops_kmeans(n, k, d, iters):
    return 2 * n * k * d + iters * (2 * n * k * d + 2 * n * k + 2 * n * d)


# ----------------------------------------------------------------------------
# synthetic inputs shared by tests and bench (bf16-representable float64)
# ----------------------------------------------------------------------------
def round_to_bf16(x):
    """Round float64/float32 values to the nearest bf16 (ties-to-even) and return
    them as float64 — so the oracle and the bf16 GPU path see identical numbers."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(F64)


def blob_tokens(n, d, blobs, sigma, rng, center_scale=1.0):
    """[ref: analysis.py:86-104] — same draw order as the reference generator."""
    centres = rng.normal(size=(blobs, d)) * center_scale
    labels = rng.permutation(np.resize(np.arange(blobs), n))
    return centres[labels] + sigma * rng.normal(size=(n, d)), labels


def blob_instance(n_q, n_k, d, q_blobs, k_blobs, sigma, seed):
    """[ref: analysis.py:107-118]"""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(7,)))
    q, _ = blob_tokens(n_q, d, q_blobs, sigma, rng)
    k, lab = blob_tokens(n_k, d, k_blobs, sigma, rng)
    vc = rng.normal(size=(k_blobs, d))
    v = vc[lab] + sigma * rng.normal(size=(n_k, d))
    return q, k, v
