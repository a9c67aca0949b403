"""The drop-in operator: svg_ear_attention(q, k, v, n_q_clusters, n_k_clusters, budget).

Per (batch, head) instance this is exactly the reference's four-call composition
    prepare -> build_error_table -> route_error_aware(global density) -> sparse_attend
(README.md:94-98, cli.py:119-134) followed by inverse_permute_rows, executed by ONE C-ABI call
(svgear_forward) on the current CUDA stream.
"""

from __future__ import annotations

import os

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._tensors import ShapeError, require_cuda, stream_ptr, workspace
from .analysis import side_seeds
from .clustering import SEED_OVERSAMPLE, reference_start, strided_start
from .router import _OVERSHOOT, entry_capacity

_EST = {"valueAware": _lib.EST_VALUE_AWARE, "plain": _lib.EST_PLAIN}


_GROUP_STREAMS = {}


def _group_streams(dev, n):
    """Per-device compute streams of the head groups (created once; every tensor they touch is
    allocated on the caller's stream and the groups are joined before the operator returns)."""
    have = _GROUP_STREAMS.setdefault(dev.index, [])
    while len(have) < n:
        have.append(torch.cuda.Stream(device=dev))
    return have[:n]


def _auto_groups(bh, n_q, n_k):
    return 2 if (bh >= 16 and min(n_q, n_k) >= 16384) else 1


def _group_layout(bh, n_q, n_k, d, c_q, c_k, groups):
    """(instance bounds, per-group workspace bytes, total bytes) of a head-group split."""
    bnd = [bh * g // groups for g in range(groups + 1)]
    frac = os.environ.get("SVGEAR_GROUP_FRACTIONS")  # experiment knob: "0.3,1.0" = cumulative shares
    if frac and groups > 1:
        cum = [float(x) for x in frac.split(",")]
        if len(cum) == groups:
            bnd = [0] + [max(1, min(bh, round(bh * c))) for c in cum]
            bnd[-1] = bh
    nds = [_lib.workspace_bytes(_lib.Shape(bnd[g + 1] - bnd[g], n_q, n_k, d, c_q, c_k)) for g in range(groups)]
    if groups > 1:  # every group's slice starts 256-byte aligned
        nds = [(x + 255) // 256 * 256 for x in nds]
    return bnd, nds, sum(nds) + (256 if groups > 1 else 0)


def operator_workspace_bytes(bh, n_q, n_k, d, n_q_clusters, n_k_clusters, head_groups=None):
    """Bytes of `workspace_buffer` that let svg_ear_attention run with the given head_groups
    (None = the operator's own choice) on bh instances."""
    groups = _auto_groups(bh, n_q, n_k) if head_groups is None else int(head_groups)
    groups = max(1, min(groups, bh))
    return _group_layout(bh, n_q, n_k, d, int(n_q_clusters), int(n_k_clusters), groups)[2]


def reference_init(q, k, n_q_clusters, n_k_clusters, seed):
    """k-means++ start centres the reference would draw for `prepare(seed=...)`, for every
    instance of a [.., S, d] batch (instance index b uses seed + b): numpy's draw reproduced bit for
    bit on the device (clustering.reference_start); the host only derives the per-instance side seeds
    (analysis.py:227) and generator states.  Exact but sequential (one dependent float64 add per token
    and centre): the parity start, ~0.4 s per Wan2.2 layer, where the default device seeding takes 1.7 ms."""
    qb = q.reshape(-1, q.shape[-2], q.shape[-1]).to(torch.bfloat16).contiguous()
    kb = k.reshape(-1, k.shape[-2], k.shape[-1]).to(torch.bfloat16).contiguous()
    seeds = [side_seeds(seed + b) for b in range(qb.shape[0])]
    return (reference_start(qb, n_q_clusters, [s_[0] for s_ in seeds]),
            reference_start(kb, n_k_clusters, [s_[1] for s_ in seeds]))


def svg_ear_attention(q, k, v, n_q_clusters, n_k_clusters, budget, *, seed=0, q_init=None,
                      k_init=None, init="device", kmeans_iters=25, estimator="valueAware",
                      overshoot="fillRemainder", single_item_fallback=True, check_fp32=False,
                      return_aux=False, workspace_buffer=None, budget_mode="globalDensity",
                      head_groups=None, stagger_groups=False, head_offset=0, total_heads=None, _row_base=0):
    """SVG-EAR attention.

    q, k, v : bf16 CUDA tensors [B, H, S, d] (or [H, S, d] / [S, d]); d in {64, 128}.
    n_q_clusters, n_k_clusters : cluster counts C_q, C_k.
    budget : exact-compute budget = global density rho in [0, 1]
             (router.DensityBudget.global_density, router.py:59-61); with
             budget_mode="perClusterTopP" it is the per-query-cluster score mass p in (0, 1]
             (router.DensityBudget.top_p, router.py:63-65 — the paper's production setting p=0.85).
    init   : "device" (default) -> k-means++ on a strided subsample, on the device, inside the one
             C-ABI call; "reference" -> the k-means++ centres the reference draws from `seed`
             (numpy's PCG64 draw reproduced bit for bit on the device, svgear_kmeans_seed_reference) —
             the parity switch: exact at any scale but sequential (~0.4 s per Wan2.2 layer);
             "strided" -> evenly strided tokens; ignored for a side whose q_init / k_init
             ([.., C, d] float32 centres) is given.
    seed   : instance (b, h) of a [B, H, S, d] call is seeded by `seed + g` with the GLOBAL
             instance index g = b * total_heads + head_offset + h.
    head_offset, total_heads : for a caller that holds only heads [head_offset, head_offset + H)
             of a layer with total_heads heads (head-parallel sharding): makes g, and with it every
             result, independent of how the heads are split.  Default: the call holds all heads.
    check_fp32 : run the executor in fp32 on CUDA cores and return a float32 output.
    head_groups : split the B*H instances into this many contiguous groups and run one
             svgear_forward per group on its own CUDA stream (joined before returning): the
             latency-bound phases of one group (late Lloyd iterations, routing) overlap the
             throughput-bound phases of another.  Results are bit-identical for every value.
             None -> 2 groups for large batches (>= 16 instances of >= 16k tokens), else 1.
    stagger_groups : group g + 1 starts when group g has finished its k-means (an event recorded
             inside svgear_forward), so its latency-bound clustering runs under group g's attention
             kernel instead of next to group g's clustering.  Same results either way; measured
             SLOWER at the Wan2.2 shape (46.8 vs 45.0 ms: the chain of small clustering kernels
             queues behind 0.3 ms attention CTAs on every SM), hence off by default.
    Returns (out, mask) — out [.., S, d] in ORIGINAL token order, mask [.., C_q, C_k] bool
    (True = block computed exactly) — plus a dict of intermediates when return_aux=True.
    """
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor")
        if t.ndim not in (2, 3, 4):
            raise ShapeError(f"{name} must be [B,H,S,d], [H,S,d] or [S,d], got shape {tuple(t.shape)}")
    if k.shape != v.shape:
        raise ValueError(f"key/value row counts differ: {tuple(k.shape)} vs {tuple(v.shape)}")
    if q.shape[:-2] != k.shape[:-2] or q.shape[-1] != k.shape[-1]:
        raise ShapeError(f"q {tuple(q.shape)} and k {tuple(k.shape)} disagree on batch/head/d")
    n_q, n_k, d = q.shape[-2], k.shape[-2], q.shape[-1]
    if d not in (64, 128):
        raise ShapeError(f"head dimension must be 64 or 128 on the B200 path, got {d}")
    for name, c, n in (("n_q_clusters", n_q_clusters, n_q), ("n_k_clusters", n_k_clusters, n_k)):
        if c < 1:
            raise ValueError(f"num_clusters must be >= 1, got {c} ({name})")
        if c > n:
            raise ValueError(f"num_clusters ({c}) exceeds token count ({n}) ({name})")
    if budget_mode not in ("globalDensity", "perClusterTopP"):
        raise ValueError(f"unknown budget mode {budget_mode!r}")
    if budget_mode == "perClusterTopP":
        if budget is None or not (0.0 < float(budget) <= 1.0):
            raise ValueError(f"perClusterTopP budget needs p in (0, 1], got {budget}")
    elif budget is None or not (0.0 <= float(budget) <= 1.0):
        raise ValueError(f"globalDensity budget needs rho in [0, 1], got {budget}")
    if kmeans_iters < 1:
        raise ValueError(f"max_iters must be >= 1, got {kmeans_iters}")
    if estimator not in _EST:
        raise ValueError(f"unknown estimator mode {estimator!r}")
    if overshoot not in _OVERSHOOT:
        raise ValueError(f"unknown overshoot policy {overshoot!r}")
    if init not in ("reference", "strided", "device"):
        raise ValueError(f"unknown init {init!r}")
    dev = require_cuda()
    lead = tuple(q.shape[:-2])
    bh = int(np.prod(lead)) if lead else 1
    h_local = lead[-1] if lead else 1
    total_heads = h_local if total_heads is None else int(total_heads)
    head_offset = int(head_offset)
    if head_offset < 0 or head_offset + h_local > total_heads:
        raise ValueError(f"heads [{head_offset}, {head_offset + h_local}) do not fit in total_heads={total_heads}")
    if len(lead) == 2 and lead[0] > 1 and total_heads != h_local:
        # the global instance indices of a head shard are contiguous per batch row only
        rows = [svg_ear_attention(
            q[b], k[b], v[b], n_q_clusters, n_k_clusters, budget, seed=seed, _row_base=b * total_heads,
            q_init=None if q_init is None else q_init[b], k_init=None if k_init is None else k_init[b],
            init=init, kmeans_iters=kmeans_iters, estimator=estimator, overshoot=overshoot,
            single_item_fallback=single_item_fallback, check_fp32=check_fp32, return_aux=return_aux,
            budget_mode=budget_mode, head_groups=head_groups, stagger_groups=stagger_groups,
            head_offset=head_offset, total_heads=total_heads) for b in range(lead[0])]
        stacked = tuple(torch.stack([r[i] for r in rows]) for i in range(2))
        if not return_aux:
            return stacked
        return stacked + ({name: torch.stack([r[2][name] for r in rows]) for name in rows[0][2]},)
    first_instance = int(_row_base) + head_offset  # global index of this call's first instance
    qb = q.to(dev, torch.bfloat16).reshape(bh, n_q, d).contiguous()
    kb = k.to(dev, torch.bfloat16).reshape(bh, n_k, d).contiguous()
    vb = v.to(dev, torch.bfloat16).reshape(bh, n_k, d).contiguous()
    c_q, c_k = int(n_q_clusters), int(n_k_clusters)

    # start centres: given, or drawn on the device INSIDE the forward call (each side's seeding on the
    # stream of its own Lloyd loop), or — parity switch — the reference's host-side draw
    seeded = False
    if q_init is None and k_init is None and init == "device":
        for c, n in ((c_q, n_q), (c_k, n_k)):
            if min(n, SEED_OVERSAMPLE * c, 4096) < c:
                raise ValueError(f"device seeding cannot hold {c} clusters in its subsample (n={n}); pass init centres")
        seeded = True
        q_init = torch.empty((bh, c_q, d), dtype=torch.float32, device=dev)
        k_init = torch.empty((bh, c_k, d), dtype=torch.float32, device=dev)
    if q_init is None or k_init is None:
        if init == "reference":
            rq, rk = reference_init(qb, kb, c_q, c_k, seed + first_instance)
        elif init == "device":
            from .clustering import device_start_pair
            rq, rk = device_start_pair(qb, c_q, kb, c_k, seed, first_instance=first_instance)
        else:
            rq, rk = strided_start(qb, c_q), strided_start(kb, c_k)
        q_init = rq if q_init is None else q_init
        k_init = rk if k_init is None else k_init
    q_init = q_init.to(dev, torch.float32).reshape(bh, c_q, d).contiguous()
    k_init = k_init.to(dev, torch.float32).reshape(bh, c_k, d).contiguous()

    if head_groups is None:
        head_groups = _auto_groups(bh, n_q, n_k)
    groups = max(1, min(int(head_groups), bh))
    layout = lambda g_count: _group_layout(bh, n_q, n_k, d, c_q, c_k, g_count)
    bounds, needs, need = layout(groups)
    if workspace_buffer is not None and groups > 1 and workspace_buffer.numel() * workspace_buffer.element_size() < need:
        groups = 1  # a caller-sized buffer for the unsplit call: run unsplit rather than fail
        bounds, needs, need = layout(1)
    ws = workspace_buffer if workspace_buffer is not None else workspace(need, dev)
    if ws.numel() * ws.element_size() < need:
        raise ValueError(f"workspace_buffer too small: need {need} bytes")
    ws_base = (ws.data_ptr() + 255) // 256 * 256 if groups > 1 else ws.data_ptr()
    out = torch.empty((bh, n_q, d), dtype=torch.float32 if check_fp32 else torch.bfloat16, device=dev)
    mask = torch.empty((bh, c_q, c_k), dtype=torch.uint8, device=dev)
    aux_t = {}
    if return_aux:
        i32, f32 = torch.int32, torch.float32
        aux_t = dict(
            q_assign=torch.empty((bh, n_q), dtype=i32, device=dev),
            k_assign=torch.empty((bh, n_k), dtype=i32, device=dev),
            q_perm=torch.empty((bh, n_q), dtype=i32, device=dev),
            k_perm=torch.empty((bh, n_k), dtype=i32, device=dev),
            q_sizes=torch.empty((bh, c_q), dtype=i32, device=dev),
            k_sizes=torch.empty((bh, c_k), dtype=i32, device=dev),
            q_offsets=torch.empty((bh, c_q), dtype=i32, device=dev),
            k_offsets=torch.empty((bh, c_k), dtype=i32, device=dev),
            q_centroids=torch.empty((bh, c_q, d), dtype=f32, device=dev),
            k_centroids=torch.empty((bh, c_k, d), dtype=f32, device=dev),
            v_centroids=torch.empty((bh, c_k, d), dtype=f32, device=dev),
            q_iters=torch.zeros((bh,), dtype=i32, device=dev),
            k_iters=torch.zeros((bh,), dtype=i32, device=dev),
            error_table=torch.empty((bh, c_q, c_k), dtype=torch.float64, device=dev),
            stabilizers=torch.empty((bh, c_q), dtype=f32, device=dev),
            mask_entries=torch.zeros((bh,), dtype=torch.int64, device=dev),
            lse=torch.empty((bh, n_q), dtype=f32, device=dev),
        )
    fn = "svgear_forward_seeded" if seeded else "svgear_forward"
    capacity = 0 if budget_mode == "perClusterTopP" else entry_capacity(float(budget), n_q * n_k)

    def launch(a, b, ws_ptr, ws_bytes, done_event=None):
        """svgear_forward for instances [a, b) on the current stream."""
        row = lambda t: t.data_ptr() + a * t.stride(0) * t.element_size()
        aux_g = None
        if return_aux or done_event is not None:
            aux_g = _lib.Aux(**({name: row(aux_t[name]) for name in _lib.Aux.FIELDS} if return_aux else {}))
            if done_event is not None:
                aux_g.kmeans_done_event = done_event.cuda_event
        head = (row(q_init), row(k_init))
        if seeded:
            head = (SEED_OVERSAMPLE, int(seed) & 0xFFFFFFFF, first_instance + a) + head
        shape_g = _lib.Shape(b - a, n_q, n_k, d, c_q, c_k)
        rc = getattr(_lib.lib(), fn)(
            C.byref(shape_g), row(qb), row(kb), row(vb), *head, int(kmeans_iters), _EST[estimator], capacity,
            _OVERSHOOT[overshoot], 1 if single_item_fallback else 0,
            _lib.EXEC_FP32_CHECK if check_fp32 else _lib.EXEC_BF16_TENSOR,
            float(budget) if budget_mode == "perClusterTopP" else 0.0, row(out), row(mask),
            C.byref(aux_g) if aux_g is not None else None, ws_ptr, ws_bytes, stream_ptr())
        _lib.check(fn, rc)

    if groups == 1:
        launch(0, bh, ws.data_ptr(), ws.numel() * ws.element_size())
    else:
        cur = torch.cuda.current_stream(dev)
        streams = _group_streams(dev, groups)
        off = ws_base
        prev_done = None
        for g in range(groups):
            streams[g].wait_stream(cur)
            if prev_done is not None:
                streams[g].wait_event(prev_done)
            done = None
            with torch.cuda.stream(streams[g]):
                if stagger_groups and g + 1 < groups:
                    done = torch.cuda.Event()
                    done.record(streams[g])  # creates the handle; re-recorded inside the call
                launch(bounds[g], bounds[g + 1], off, needs[g], done)
            prev_done = done
            off += needs[g]
        for g in range(groups):
            cur.wait_stream(streams[g])
    out = out.reshape(*lead, n_q, d)
    mask_b = mask.bool().reshape(*lead, c_q, c_k)
    if not return_aux:
        return out, mask_b
    aux = {name: t.reshape(tuple(lead) + tuple(t.shape[1:])) for name, t in aux_t.items()}
    aux["q_init"], aux["k_init"] = q_init.reshape(*lead, c_q, d), k_init.reshape(*lead, c_k, d)
    return out, mask_b, aux
