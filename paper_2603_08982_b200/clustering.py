"""GPU k-means + cluster-contiguous permutation — host mirror of routedattn.clustering.

Same names and argument meaning as the reference (clustering.py:144-257); arrays are torch CUDA
tensors.  `kmeans` accepts one instance [n, d] (as the reference) or a batch [bh, n, d].
`kmeans` (the reference's entry point, seed-faithful) starts from the reference's own k-means++
centres for a given `seed` (clustering.py:65-84, 178-180): `reference_start` reproduces numpy's draw
bit for bit on the device (svgear_kmeans_seed_reference); `seeded_start` is the same draw in host numpy,
kept as the cross-check of the tests; `device_start` is the fast device-side seeding the operator uses.
Lloyd iterations, repair, permutation and means run in libsvgear (svgear_kmeans).
"""

from __future__ import annotations

import ctypes as C
from ctypes import c_size_t as _SZ
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._tensors import ShapeError, as_f32, as_tokens, stream_ptr, workspace


@dataclass(frozen=True)
class ClusterModel:
    """Result of clustering (clustering.py:29-39).  Tensors live on the GPU; a model fitted on a
    batch keeps the leading [bh] dimension on every field."""

    num_clusters: int
    assignments: torch.Tensor  # (n,) int32, raw token order
    centroids: torch.Tensor    # (num_clusters, d) float32
    sizes: torch.Tensor        # (num_clusters,) int32, all >= 1
    permutation: torch.Tensor  # (n,) int32; permuted[i] = tokens[permutation[i]]
    offsets: torch.Tensor      # (num_clusters,) int32
    flops: int = 0
    iters: object = None       # Lloyd iterations executed (int, or tensor for a batch)
    inertia: object = None


def kmeans_pp_init(tokens, k, rng):
    """k-means++ centres with the reference's draw sequence (clustering.py:65-84), float64 numpy."""
    x = np.ascontiguousarray(tokens, dtype=np.float64)
    n = x.shape[0]
    centres = np.empty((k, x.shape[1]), dtype=np.float64)
    taken = np.zeros(n, dtype=bool)
    i = int(rng.integers(n))
    centres[0] = x[i]
    taken[i] = True
    near = ((x - centres[0]) ** 2).sum(axis=1)
    for c in range(1, k):
        tot = near.sum()
        i = int(rng.choice(n, p=near / tot)) if tot > 0.0 else int(np.flatnonzero(~taken)[0])
        centres[c] = x[i]
        taken[i] = True
        near = np.minimum(near, ((x - centres[c]) ** 2).sum(axis=1))
    return centres


def seeded_start(tokens, k, seed, restart=0):
    """Start centres of restart `restart` for `seed` (clustering.py:178-180)."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(restart,)))
    return kmeans_pp_init(tokens, k, rng)


def pcg64_states(seeds, restart=0):
    """PCG64 states {state_hi, state_lo, inc_hi, inc_lo} of the generators the reference creates for
    `seeds` (clustering.py:178-180): numpy.random.PCG64(SeedSequence(entropy=seed, spawn_key=(restart,))).
    Host side: SeedSequence hashing is a few integer operations; everything after it runs on the device."""
    out = np.empty((len(seeds), 4), dtype=np.uint64)
    lo64 = (1 << 64) - 1
    for i, seed in enumerate(seeds):
        st = np.random.PCG64(np.random.SeedSequence(entropy=int(seed), spawn_key=(int(restart),))).state["state"]
        out[i] = (st["state"] >> 64, st["state"] & lo64, st["inc"] >> 64, st["inc"] & lo64)
    return out


def reference_start(tokens, k, seeds, restart=0, return_picks=False):
    """The reference's k-means++ start centres (clustering._kmeans_pp_init under numpy's PCG64,
    clustering.py:65-84, 178-180) computed ON THE DEVICE, bit-identical to `seeded_start` on the host
    (svgear_kmeans_seed_reference: numpy's float64 operation order and RNG reproduced exactly).
    tokens [bh, n, d] (or [n, d]) bf16 CUDA; seeds: one side seed per instance."""
    x = (tokens if tokens.ndim == 3 else tokens.unsqueeze(0)).contiguous()
    bh, n, d = x.shape
    seeds = [int(seeds)] if np.isscalar(seeds) else [int(s_) for s_ in seeds]
    if len(seeds) != bh:
        raise ValueError(f"got {len(seeds)} seeds for {bh} instances")
    states = torch.from_numpy(pcg64_states(seeds, restart).view(np.int64)).to(x.device)
    out = torch.empty((bh, int(k), d), dtype=torch.float32, device=x.device)
    picks = torch.empty((bh, int(k)), dtype=torch.int32, device=x.device)
    need = _SZ(0)
    _lib.check("svgear_kmeans_seed_reference_workspace",
               _lib.lib().svgear_kmeans_seed_reference_workspace(bh, n, C.byref(need)))
    ws = workspace(int(need.value), x.device)
    rc = _lib.lib().svgear_kmeans_seed_reference(bh, n, d, int(k), x.data_ptr(), states.data_ptr(), out.data_ptr(),
                                                 picks.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_kmeans_seed_reference", rc)
    res = out if tokens.ndim == 3 else out[0]
    return (res, picks if tokens.ndim == 3 else picks[0]) if return_picks else res


def strided_start(tokens, k):
    """Deterministic device-side start: k evenly strided tokens.  NOT the reference's seeding —
    used when no seed-faithful start is needed (benchmarks, warm-up of a centroid cache)."""
    n = tokens.shape[-2]
    idx = torch.div(torch.arange(k, device=tokens.device) * n, k, rounding_mode="floor")
    return tokens.index_select(-2, idx).float().contiguous()


SEED_OVERSAMPLE = 8  # subsample tokens per centre of the device-side seeding


def _seed_launch(x, k, seed, oversample, first_instance):
    """svgear_kmeans_seed on x [bh, n, d] bf16 -> start centres [bh, k, d] f32 (current stream)."""
    bh, n, d = x.shape
    out = torch.empty((bh, k, d), dtype=torch.float32, device=x.device)
    m = min(n, int(oversample) * k, 4096)
    if m < k:
        raise ValueError(f"device seeding needs a subsample of >= {k} tokens, got {m} (n={n}, oversample={oversample})")
    ws = workspace(bh * m * m * 2 + 256, x.device)
    rc = _lib.lib().svgear_kmeans_seed(bh, n, d, k, x.data_ptr(), int(oversample), int(seed) & 0xFFFFFFFF,
                                       int(first_instance), out.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_kmeans_seed", rc)
    return out


def device_start(tokens, k, seed=0, oversample=SEED_OVERSAMPLE, first_instance=0):
    """Device-side k-means++ start on a strided subsample (svgear_kmeans_seed: Gram matrix of the
    subsample on the tensor cores, then the D^2 rounds).  Deterministic, but NOT the reference's numpy
    draw — use `seeded_start` / init="reference" for parity runs.  Instance b of a batch draws as
    instance first_instance + b."""
    x = (tokens if tokens.ndim == 3 else tokens.unsqueeze(0)).contiguous()
    out = _seed_launch(x, int(k), seed, oversample, first_instance)
    return out if tokens.ndim == 3 else out[0]


_SIDE_STREAMS = {}


def device_start_pair(q, c_q, k, c_k, seed=0, oversample=SEED_OVERSAMPLE, first_instance=0):
    """device_start for the query and the key side on two streams: the D^2 rounds run one CTA per
    instance (c sequential rounds), so the sides overlap on disjoint SMs.  The key side draws with
    seed + 0x9E37, as svgear_forward_seeded does.  The helper stream is joined before returning."""
    xq = (q if q.ndim == 3 else q.unsqueeze(0)).contiguous()
    xk = (k if k.ndim == 3 else k.unsqueeze(0)).contiguous()
    dev = xq.device
    cur = torch.cuda.current_stream(dev)
    side = _SIDE_STREAMS.get(dev.index)
    if side is None:
        side = _SIDE_STREAMS[dev.index] = torch.cuda.Stream(device=dev)
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        ok = _seed_launch(xk, int(c_k), seed + 0x9E37, oversample, first_instance)
        ok.record_stream(cur)
    oq = _seed_launch(xq, int(c_q), seed, oversample, first_instance)
    cur.wait_stream(side)
    return (oq if q.ndim == 3 else oq[0]), (ok if k.ndim == 3 else ok[0])


def _pad_centers(tok_f32, centers, k):
    """Grow a centre set to k rows by farthest-token selection (clustering.py:87-101)."""
    centers = torch.as_tensor(centers, dtype=torch.float32, device=tok_f32.device)
    if centers.ndim != 2 or centers.shape[1] != tok_f32.shape[1]:
        raise ValueError(
            f"init centroids must be 2-D with {tok_f32.shape[1]} columns, got {tuple(centers.shape)}")
    if centers.shape[0] > k:
        raise ValueError(f"got {centers.shape[0]} init centroids for {k} clusters")
    d2 = torch.cdist(tok_f32.double(), centers.double()).pow(2).min(dim=1).values
    while centers.shape[0] < k:
        i = int(torch.argmax(d2))
        centers = torch.cat([centers, tok_f32[i:i + 1]], dim=0)
        d2 = torch.minimum(d2, (tok_f32.double() - tok_f32[i].double()).pow(2).sum(dim=1))
    return centers


def run_lloyd(x, starts, max_iters, fp32_check=False, full_eval=False, want_inertia=True):
    """x [bh,n,d] bf16, starts [bh,c,d] f32 -> dict of raw svgear_kmeans outputs.

    `full_eval` evaluates every token against every centre in every iteration; by default the
    tensor-core mode skips tokens whose distance bounds prove their cluster cannot change (same
    assignments, see SVGEAR_KMEANS_FULL_EVAL in include/svgear.h)."""
    bh, n, d = x.shape
    c = starts.shape[1]
    dev = x.device
    out = dict(
        assign=torch.empty((bh, n), dtype=torch.int32, device=dev),
        perm=torch.empty((bh, n), dtype=torch.int32, device=dev),
        sizes=torch.empty((bh, c), dtype=torch.int32, device=dev),
        offsets=torch.empty((bh, c), dtype=torch.int32, device=dev),
        centroids=torch.empty((bh, c, d), dtype=torch.float32, device=dev),
        iters=torch.zeros((bh,), dtype=torch.int32, device=dev),
        inertia=torch.zeros((bh,), dtype=torch.float64, device=dev),
    )
    shape = _lib.Shape(bh, n, n, d, c, c)
    ws = workspace(_lib.workspace_bytes(shape), dev)
    rc = _lib.lib().svgear_kmeans(
        (_lib.EXEC_FP32_CHECK if fp32_check else _lib.EXEC_BF16_TENSOR) | (_lib.KMEANS_FULL_EVAL if full_eval else 0),
        bh, n, d, c, x.data_ptr(), starts.data_ptr(), int(max_iters), out["assign"].data_ptr(),
        out["perm"].data_ptr(), out["sizes"].data_ptr(), out["offsets"].data_ptr(),
        out["centroids"].data_ptr(), out["iters"].data_ptr(), out["inertia"].data_ptr() if want_inertia else None,
        ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check("svgear_kmeans", rc)
    return out


def _flops(n, k, d, iters):
    return 2 * n * k * d + iters * (2 * n * k * d + 2 * n * k + 2 * n * d)  # clustering.py:138-140


def kmeans(tokens, num_clusters, *, max_iters=25, seed=0, restarts=1, init_centroids=None,
           fp32_check=False):
    """Cluster token rows; best of `restarts` seeded runs (+ an optional warm start).

    Mirrors clustering.kmeans (clustering.py:144-207) including its validation errors.  For a
    batch [bh, n, d], instance b is seeded with `seed + b` (or `seed[b]` when a list of per-instance
    seeds is given) and `init_centroids` may be [bh, c', d].
    """
    x, was_2d = _validated(tokens, num_clusters, restarts, max_iters)
    bh, n, d = x.shape
    k = int(num_clusters)
    seeds = [int(s_) for s_ in seed] if isinstance(seed, (list, tuple)) else [int(seed) + b for b in range(bh)]
    if len(seeds) != bh:
        raise ValueError(f"got {len(seeds)} seeds for {bh} instances")
    pool = []  # list over starts of [bh,k,d] f32: the reference's seeded draws, reproduced on the device
    for r in range(restarts):
        pool.append(reference_start(x, k, seeds, r))
    if init_centroids is not None:
        ic = torch.as_tensor(np.asarray(init_centroids) if not isinstance(init_centroids, torch.Tensor)
                             else init_centroids)
        if ic.ndim == 2:
            ic = ic.unsqueeze(0).expand(bh, -1, -1)
        xf = x.float()
        pool.append(torch.stack([_pad_centers(xf[b], ic[b], k) for b in range(bh)]))
    # every start is one more batch instance: [S*bh, ...]
    S = len(pool)
    res = run_lloyd(x.repeat(S, 1, 1) if S > 1 else x, torch.cat(pool, dim=0).contiguous(), max_iters,
                    fp32_check=fp32_check)
    inertia = res["inertia"].view(S, bh)
    best = torch.argmin(inertia, dim=0)  # ties -> earliest start, as the reference
    pick = best * bh + torch.arange(bh, device=x.device)
    iters = res["iters"].view(S, bh)
    flops = int(sum(_flops(n, k, d, int(i)) for i in iters.flatten().tolist()))
    fields = {key: res[key].index_select(0, pick) for key in ("assign", "perm", "sizes", "offsets", "centroids")}
    sq = (lambda t: t[0]) if was_2d else (lambda t: t)
    it = iters.gather(0, best.unsqueeze(0))[0]
    return ClusterModel(
        num_clusters=k, assignments=sq(fields["assign"]), centroids=sq(fields["centroids"]),
        sizes=sq(fields["sizes"]), permutation=sq(fields["perm"]), offsets=sq(fields["offsets"]),
        flops=flops, iters=int(it[0]) if was_2d else it,
        inertia=float(inertia.min(dim=0).values[0]) if was_2d else inertia.min(dim=0).values)


def _validated(tokens, num_clusters, restarts, max_iters):
    if isinstance(tokens, torch.Tensor):
        nd, n = tokens.ndim, (tokens.shape[-2] if tokens.ndim >= 2 else 0)
    else:
        arr = np.asarray(tokens)
        nd, n = arr.ndim, (arr.shape[-2] if arr.ndim >= 2 else 0)
    if nd not in (2, 3):
        raise ShapeError(f"token matrix must be 2-D, got shape {tuple(np.shape(tokens))}")
    if num_clusters < 1:
        raise ValueError(f"num_clusters must be >= 1, got {num_clusters}")
    if num_clusters > n:
        raise ValueError(f"num_clusters ({num_clusters}) exceeds token count ({n})")
    if restarts < 1:
        raise ValueError(f"restarts must be >= 1, got {restarts}")
    if max_iters < 1:
        raise ValueError(f"max_iters must be >= 1, got {max_iters}")
    return as_tokens(tokens)


def permute_rows(tokens, model: ClusterModel):
    """Reorder raw-order rows into cluster-contiguous order (clustering.py:210-212)."""
    x, was_2d = as_tokens(tokens, check_finite=False)
    bh, n, d = x.shape
    perm = model.permutation.view(bh, n).contiguous()
    out = torch.empty_like(x)
    rc = _lib.lib().svgear_permute_rows(bh, n, d, x.data_ptr(), perm.data_ptr(), out.data_ptr(), stream_ptr())
    _lib.check("svgear_permute_rows", rc)
    return out[0] if was_2d else out


def inverse_permute_rows(rows, model: ClusterModel):
    """Undo permute_rows (clustering.py:215-219): out[perm[i]] = rows[i]."""
    perm = model.permutation.long()
    out = torch.empty_like(rows)
    if perm.ndim == 1:
        out[perm] = rows
    else:
        out.scatter_(1, perm.unsqueeze(-1).expand_as(rows) if rows.ndim == 3 else perm, rows)
    return out


def segment_means(tokens_permuted, model: ClusterModel):
    """Per-cluster means of a cluster-contiguous matrix (clustering.py:247-257), float32."""
    x, was_2d = as_tokens(tokens_permuted, check_finite=False)
    bh, n, d = x.shape
    c = model.num_clusters
    sizes = model.sizes.view(bh, c).contiguous()
    offsets = model.offsets.view(bh, c).contiguous()
    out = torch.empty((bh, c, d), dtype=torch.float32, device=x.device)
    rc = _lib.lib().svgear_segment_means(bh, n, d, c, x.data_ptr(), sizes.data_ptr(), offsets.data_ptr(),
                                         out.data_ptr(), stream_ptr())
    _lib.check("svgear_segment_means", rc)
    return out[0] if was_2d else out


def cluster_means(model: ClusterModel, tokens):
    """Per-cluster means of raw-order `tokens` under the model (clustering.py:222-240)."""
    n = model.assignments.shape[-1]
    if tokens.shape[-2] != n:
        raise ValueError(f"token count {tokens.shape[-2]} does not match model ({n} assignments)")
    return segment_means(permute_rows(tokens, model), model)
