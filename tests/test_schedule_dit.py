"""SURVEY §8 rows f2 (warm-up schedule, warm-started k-means across denoising steps) and f3 (the
DiT attention block around the operator).  CPU tests cover the schedule logic and argument
validation; GPU tests compare the warm-started operator with the oracle's Lloyd from the same
centres (bit-exact permutations and masks) and the two layout kernels with a torch fp32 reference
(tolerance: one bf16 rounding of an fp32 result, 2^-8 relative per element)."""

import numpy as np
import pytest
import torch

import paper_2603_08982_b200 as P
from paper_2603_08982_b200 import dit, schedule
from oracle import svgear_oracle as O


# ------------------------------------------------------------------------------------------------
# host logic (CPU)
# ------------------------------------------------------------------------------------------------
class TestWarmupSchedule:
    def test_wan22_counts(self):
        s = schedule.WarmupSchedule.wan22()  # PAPER.md Table `config`: time-warm 10/50, layer-warm 1/40
        assert s.sparse_calls == 40 * 39
        assert s.dense_calls == 50 * 40 - 40 * 39
        assert sum(s.is_dense(l, t) for l in range(40) for t in range(50)) == s.dense_calls

    def test_dense_region(self):
        s = schedule.WarmupSchedule(total_steps=6, time_warm=2, total_layers=3, layer_warm=1)
        dense = {(l, t) for l in range(3) for t in range(6) if s.is_dense(l, t)}
        assert dense == {(l, t) for l in range(3) for t in range(6) if t < 2 or l < 1}

    def test_none(self):
        s = schedule.WarmupSchedule.none(4, 2)
        assert s.dense_calls == 0 and not s.is_dense(0, 0)

    @pytest.mark.parametrize("kw", [dict(total_steps=0), dict(time_warm=-1), dict(time_warm=51),
                                    dict(layer_warm=41), dict(total_layers=0)])
    def test_rejects_bad_values(self, kw):
        with pytest.raises(ValueError):
            schedule.WarmupSchedule(**kw)

    def test_index_errors(self):
        s = schedule.WarmupSchedule.wan22()
        with pytest.raises(IndexError):
            s.is_dense(40, 0)
        with pytest.raises(IndexError):
            s.is_dense(0, 50)

    def test_stack_plan_without_state(self):
        st = schedule.SvgEarStack(8, 12, 0.25, schedule=schedule.WarmupSchedule(4, 1, 2, 1))
        assert st.plan(0, 3) == "dense" and st.plan(1, 0) == "dense" and st.plan(1, 1) == "cold"
        with pytest.raises(ValueError):
            schedule.SvgEarStack(8, 12, 0.25, warm_iters=0)


class TestDitHostLogic:
    def test_rope_table_matches_direct_formula(self):
        t, hh, w, d = 3, 4, 5, 128
        cos, sin = dit.rope_table_3d((t, hh, w), d)
        assert cos.shape == (60, 64) and sin.shape == (60, 64)
        n_hw = 64 // 3
        n_t = 64 - 2 * n_hw
        tok = (2 * hh + 3) * w + 4  # (t=2, h=3, w=4)
        ang = np.concatenate([2 * 10000.0 ** (-np.arange(n_t) / n_t), 3 * 10000.0 ** (-np.arange(n_hw) / n_hw),
                              4 * 10000.0 ** (-np.arange(n_hw) / n_hw)])
        np.testing.assert_allclose(cos[tok].numpy(), np.cos(ang), atol=1e-6)
        np.testing.assert_allclose(sin[tok].numpy(), np.sin(ang), atol=1e-6)
        assert torch.all(cos[0] == 1) and torch.all(sin[0] == 0)

    def test_argument_errors_come_before_the_device_check(self):
        x = torch.zeros(1, 4, 3 * 2 * 64, dtype=torch.bfloat16)
        with pytest.raises(ValueError):
            dit.qkv_prologue(x, 2, norm="layer")
        with pytest.raises(P.ShapeError):
            dit.qkv_prologue(torch.zeros(1, 4, 100, dtype=torch.bfloat16), 2)
        with pytest.raises(P.ShapeError):
            dit.qkv_prologue(torch.zeros(1, 4, 3 * 2 * 32, dtype=torch.bfloat16), 2)
        with pytest.raises(P.ShapeError):
            dit.heads_to_tokens(torch.zeros(2, 4, 64))
        with pytest.raises(P.ShapeError):
            dit.SvgEarSelfAttention(100, 3)

    @pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
    def test_no_cpu_fallback(self):
        x = torch.zeros(1, 4, 3 * 2 * 64, dtype=torch.bfloat16)
        with pytest.raises(RuntimeError):
            dit.qkv_prologue(x, 2)
        with pytest.raises(RuntimeError):
            dit.heads_to_tokens(torch.zeros(1, 2, 4, 64, dtype=torch.bfloat16))


# ------------------------------------------------------------------------------------------------
# GPU
# ------------------------------------------------------------------------------------------------
def _prologue_reference(qkv, h, d, norm, wq, wk, eps, rope, rope_mode):
    """torch fp32 restatement of svgear_qkv_prologue."""
    b, s = qkv.shape[:2]
    x = qkv.float().reshape(b, s, 3, h, d)
    outs = []
    for op, w in ((0, wq), (1, wk)):
        y = x[:, :, op]
        if norm == "head":
            y = y * torch.rsqrt((y * y).mean(-1, keepdim=True) + eps) * w.reshape(h, d)
        elif norm == "token":
            y = y * torch.rsqrt((y * y).mean((-2, -1), keepdim=True) + eps) * w.reshape(h, d)
        if rope is not None:
            cos, sin = rope
            L = cos.shape[0]
            z = y[:, :L]
            c, sn = cos[None, :, None, :], sin[None, :, None, :]
            if rope_mode == "interleaved":
                a, bb = z[..., 0::2], z[..., 1::2]
                r = torch.stack([a * c - bb * sn, bb * c + a * sn], dim=-1).reshape(z.shape)
            else:
                a, bb = z[..., : d // 2], z[..., d // 2:]
                r = torch.cat([a * c - bb * sn, bb * c + a * sn], dim=-1)
            y = torch.cat([r, y[:, L:]], dim=1)
        outs.append(y.permute(0, 2, 1, 3))
    outs.append(x[:, :, 2].permute(0, 2, 1, 3))
    return outs


@pytest.mark.gpu
class TestQkvPrologue:
    @pytest.mark.parametrize("d", [64, 128])
    @pytest.mark.parametrize("norm", ["none", "head", "token"])
    @pytest.mark.parametrize("rope_mode", [None, "interleaved", "half_split"])
    def test_against_fp32_reference(self, d, norm, rope_mode):
        g = torch.Generator(device="cuda").manual_seed(d + len(norm))
        b, s, h, text = 2, 75, 5, 11
        qkv = torch.randn(b, s, 3 * h * d, generator=g, device="cuda").to(torch.bfloat16)
        wq = 1 + 0.1 * torch.randn(h * d, generator=g, device="cuda")
        wk = 1 + 0.1 * torch.randn(h * d, generator=g, device="cuda")
        rope = None
        if rope_mode is not None:
            cos, sin = dit.rope_table_3d((4, 4, 4), d, device="cuda")  # 64 video tokens + 11 text tokens
            assert cos.shape[0] == s - text
            rope = (cos, sin)
        q, k, v = dit.qkv_prologue(qkv, h, norm=norm, q_weight=wq, k_weight=wk, eps=1e-6, rope=rope,
                                   rope_mode=rope_mode or "interleaved")
        rq, rk, rv = _prologue_reference(qkv, h, d, norm, wq, wk, 1e-6, rope, rope_mode)
        assert torch.equal(v, rv.to(torch.bfloat16))
        for got, ref in ((q, rq), (k, rk)):
            assert got.shape == (b, h, s, d) and got.dtype == torch.bfloat16
            err = (got.float() - ref).abs()
            assert bool((err <= 2.0 ** -8 * ref.abs() + 1e-6).all()), float(err.max())

    def test_wide_token(self):  # Wan2.2 width: 40 heads x 128 = 5120 (three chunks per thread)
        g = torch.Generator(device="cuda").manual_seed(3)
        b, s, h, d = 1, 33, 40, 128
        qkv = torch.randn(b, s, 3, h, d, generator=g, device="cuda").to(torch.bfloat16)
        w = torch.ones(h * d, device="cuda")
        rope = dit.rope_table_3d((1, 3, 11), d, device="cuda")
        q, k, v = dit.qkv_prologue(qkv, h, norm="token", q_weight=w, k_weight=w, rope=rope)
        rq, rk, rv = _prologue_reference(qkv.reshape(b, s, -1), h, d, "token", w, w, 1e-6, rope, "interleaved")
        assert torch.equal(v, rv.to(torch.bfloat16))
        for got, ref in ((q, rq), (k, rk)):
            assert bool(((got.float() - ref).abs() <= 2.0 ** -8 * ref.abs() + 1e-6).all())

    @pytest.mark.parametrize("d", [64, 128])
    def test_heads_to_tokens_is_a_pure_transpose(self, d):
        x = torch.randn(2, 7, 301, d, device="cuda").to(torch.bfloat16)
        out = dit.heads_to_tokens(x)
        assert torch.equal(out, x.permute(0, 2, 1, 3).reshape(2, 301, 7 * d))

    def test_c_abi_rejects_bad_arguments(self):
        from paper_2603_08982_b200 import _lib
        L = _lib.lib()
        buf = torch.zeros(1 << 16, dtype=torch.uint8, device="cuda")
        p = buf.data_ptr()
        assert L.svgear_qkv_prologue(1, 4, 2, 64, None, 0, None, None, 0.0, 0, 0, None, None, p, p, p, None) == _lib.EINVAL
        assert L.svgear_qkv_prologue(1, 4, 2, 64, p, 3, None, None, 0.0, 0, 0, None, None, p, p, p, None) == _lib.EINVAL
        assert L.svgear_qkv_prologue(1, 4, 2, 64, p, 1, None, None, 1e-6, 0, 0, None, None, p, p, p, None) == _lib.EINVAL
        assert L.svgear_qkv_prologue(1, 4, 2, 64, p, 0, None, None, 0.0, 1, 2, None, None, p, p, p, None) == _lib.EINVAL
        assert L.svgear_qkv_prologue(1, 4, 2, 96, p, 0, None, None, 0.0, 0, 0, None, None, p, p, p, None) == _lib.ESHAPE
        assert L.svgear_qkv_prologue(1, 4, 80, 128, p, 0, None, None, 0.0, 0, 0, None, None, p, p, p, None) == _lib.ESHAPE
        assert L.svgear_heads_to_tokens(1, 4, 2, 32, p, p, None) == _lib.ESHAPE
        assert L.svgear_heads_to_tokens(1, 4, 2, 64, None, p, None) == _lib.EINVAL


def _drifted_instances(S, d, cq, ck, steps, H, drift=0.03, sigma=0.1):
    """Per head a fixed blob mixture whose centres random-walk from step to step (bf16-rounded)."""
    out = []
    for h in range(H):
        rng = np.random.default_rng(100 + h)
        qc, kc, vc = rng.normal(size=(cq, d)), rng.normal(size=(ck, d)), rng.normal(size=(ck, d))
        ql, kl = rng.integers(cq, size=S), rng.integers(ck, size=S)
        seq = []
        for _ in range(steps):
            qc, kc, vc = (c + drift * rng.normal(size=c.shape) for c in (qc, kc, vc))
            seq.append(tuple(O.round_to_bf16(c[l] + sigma * rng.normal(size=(S, d)))
                             for c, l in ((qc, ql), (kc, kl), (vc, kl))))
        out.append(seq)
    return out


@pytest.mark.gpu
class TestStackWarmStart:
    def test_warm_started_steps_match_the_oracle_lloyd_from_the_same_centres(self):
        S, d, cq, ck, rho, H, steps, warm_iters = 640, 64, 8, 12, 0.25, 2, 3, 3
        data = _drifted_instances(S, d, cq, ck, steps, H)
        stack = schedule.SvgEarStack(cq, ck, rho, schedule=schedule.WarmupSchedule.none(steps, 1),
                                     warm_iters=warm_iters, init="reference")
        prev = None
        for t in range(steps):
            q, k, v = (torch.from_numpy(np.stack([data[h][t][i] for h in range(H)])).to("cuda", torch.bfloat16)
                       .unsqueeze(0) for i in range(3))
            assert stack.plan(0, t) == ("cold" if t == 0 else "warm")
            out, mask = stack.attend(0, t, q, k, v, return_mask=True)
            st = stack._layers[(0, 0)]
            for h in range(H):
                if t == 0:
                    ref = O.forward(*data[h][t], cq, ck, rho, seed=h)
                else:
                    ref = O.forward(*data[h][t], cq, ck, rho, max_iters=warm_iters,
                                    q_starts=[prev[0][h].astype(np.float64)],
                                    k_starts=[prev[1][h].astype(np.float64)])
                    assert int(st.q_iters[0, h]) == ref.prep.q_model.iters <= warm_iters
                    assert int(st.k_iters[0, h]) == ref.prep.k_model.iters <= warm_iters
                assert np.array_equal(mask[0, h].cpu().numpy(), ref.mask.selected)
                err = np.linalg.norm(out[0, h].float().cpu().numpy() - ref.out) / np.linalg.norm(ref.out)
                assert err <= 1e-2, err
                np.testing.assert_allclose(st.q_centroids[0, h].cpu().numpy(), ref.prep.q_model.centroids,
                                           atol=1e-5)
            prev = (st.q_centroids[0].cpu().numpy(), st.k_centroids[0].cpu().numpy())
        assert stack.calls == {"dense": 0, "cold": 1, "warm": steps - 1}

    def test_dense_steps_and_gaps(self):
        S, d, cq, ck, H = 512, 64, 8, 12, 2
        data = _drifted_instances(S, d, cq, ck, 4, H)
        stack = schedule.SvgEarStack(cq, ck, 0.25, schedule=schedule.WarmupSchedule(4, 1, 2, 1))
        for t in range(4):
            q, k, v = (torch.from_numpy(np.stack([data[h][t][i] for h in range(H)])).to("cuda", torch.bfloat16)
                       .unsqueeze(0) for i in range(3))
            for layer in range(2):
                if layer == 1 and t == 2:
                    continue  # a skipped step: the next call of this layer must start cold again
                plan = stack.plan(layer, t)
                out = stack.attend(layer, t, q, k, v)
                assert out.shape == q.shape
                if t == 0 or layer == 0:
                    assert plan == "dense"
                    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
                    assert float((out.float() - ref).norm() / ref.norm()) < 1e-2
                else:
                    assert plan == ("cold" if t in (1, 3) else "warm")
        stack.reset()
        assert stack.plan(1, 2) == "cold"

    def test_cfg_branches_keep_their_own_centroid_cache(self):
        """Classifier-free guidance calls every layer twice per step: each branch warm-starts from its
        own previous step (one cache per layer made the second call of a step cold)."""
        S, d, cq, ck, H = 512, 64, 8, 12, 2
        data = _drifted_instances(S, d, cq, ck, 3, H)
        other = _drifted_instances(S, d, cq, ck, 3, H, seed=77) if "seed" in _drifted_instances.__code__.co_varnames \
            else [[tuple(np.ascontiguousarray(a[::-1]) for a in step) for step in head] for head in data]
        stack = schedule.SvgEarStack(cq, ck, 0.25, schedule=schedule.WarmupSchedule.none(3, 1))
        solo = schedule.SvgEarStack(cq, ck, 0.25, schedule=schedule.WarmupSchedule.none(3, 1))
        for t in range(3):
            for branch, src in ((0, data), (1, other)):
                q, k, v = (torch.from_numpy(np.stack([src[h][t][i] for h in range(H)])).to("cuda", torch.bfloat16)
                           .unsqueeze(0) for i in range(3))
                assert stack.plan(0, t, branch=branch) == ("cold" if t == 0 else "warm")
                out = stack.attend(0, t, q, k, v, branch=branch)
                if branch == 0:  # the conditional branch is unaffected by the other branch's calls
                    assert torch.equal(out, solo.attend(0, t, q, k, v))
        assert stack.calls == {"dense": 0, "cold": 2, "warm": 4}


@pytest.mark.gpu
class TestDitBlock:
    def test_block_equals_its_parts(self):
        torch.manual_seed(0)
        dim, h, S = 256, 4, 512
        blk = dit.SvgEarSelfAttention(dim, h, norm="head", device="cuda")
        x = torch.randn(1, S, dim, device="cuda").to(torch.bfloat16)
        rope = dit.rope_table_3d((2, 16, 16), 64, device="cuda")
        # dense schedule: the block must agree with a torch restatement of the same block
        dense = schedule.SvgEarStack(8, 12, 0.25, schedule=schedule.WarmupSchedule(1, 1, 1, 1))
        y = blk(x, dense, 0, 0, rope=rope)
        qkv = blk.qkv(x)
        rq, rk, rv = _prologue_reference(qkv, h, 64, "head", blk.q_norm_weight, blk.k_norm_weight, blk.eps, rope,
                                         "interleaved")
        o = torch.nn.functional.scaled_dot_product_attention(rq, rk, rv)
        ref = blk.proj(o.permute(0, 2, 1, 3).reshape(1, S, dim).to(torch.bfloat16))
        assert float((y.float() - ref.float().detach()).norm() / ref.float().detach().norm()) < 2e-2
        # sparse at rho = 1 is dense attention through the SVG-EAR kernels
        full = schedule.SvgEarStack(8, 12, 1.0, schedule=schedule.WarmupSchedule.none(1, 1))
        y1 = blk(x, full, 0, 0, rope=rope)
        assert full.calls["cold"] == 1
        assert float((y1.float() - ref.float().detach()).norm() / ref.float().detach().norm()) < 2e-2


@pytest.mark.gpu
class TestStackPaperMode:
    def test_top_p_budget_through_the_stack_equals_the_operator(self):
        """The paper's production setting (perClusterTopP, p = 0.85) through SvgEarStack: a cold call is
        the operator call, a warm call is the operator call started from the cached centroids."""
        S, d, cq, ck, H = 768, 64, 8, 16, 3
        data = _drifted_instances(S, d, cq, ck, 2, H)
        stack = schedule.SvgEarStack(cq, ck, 0.85, budget_mode="perClusterTopP",
                                     schedule=schedule.WarmupSchedule.none(2, 1), warm_iters=5)
        mk = lambda t: tuple(torch.from_numpy(np.stack([data[h][t][i] for h in range(H)])).to("cuda", torch.bfloat16)
                             .unsqueeze(0) for i in range(3))
        q0, k0, v0 = mk(0)
        out0, mask0 = stack.attend(0, 0, q0, k0, v0, return_mask=True)
        ref0 = P.svg_ear_attention(q0, k0, v0, cq, ck, 0.85, budget_mode="perClusterTopP", init="device", seed=0,
                                   return_aux=True)
        assert torch.equal(out0, ref0[0]) and torch.equal(mask0, ref0[1])
        q1, k1, v1 = mk(1)
        out1, mask1 = stack.attend(0, 1, q1, k1, v1, return_mask=True)
        ref1 = P.svg_ear_attention(q1, k1, v1, cq, ck, 0.85, budget_mode="perClusterTopP", kmeans_iters=5,
                                   q_init=ref0[2]["q_centroids"], k_init=ref0[2]["k_centroids"])
        assert torch.equal(out1, ref1[0]) and torch.equal(mask1, ref1[1])
        # every query cluster keeps at least its own top-p share of key clusters exact
        assert bool(mask1.any(dim=-1).all())

    def test_hunyuan_style_block_with_text_tokens(self):
        torch.manual_seed(1)
        dim, h, video, text = 256, 2, 512, 64
        blk = dit.SvgEarSelfAttention(dim, h, norm="head", device="cuda")
        x = torch.randn(1, video + text, dim, device="cuda").to(torch.bfloat16)
        rope = dit.rope_table_3d((2, 16, 16), 128, device="cuda")  # covers the video tokens only
        dense = schedule.SvgEarStack(8, 12, 0.25, schedule=schedule.WarmupSchedule(1, 1, 1, 1))
        y = blk(x, dense, 0, 0, rope=rope)
        qkv = blk.qkv(x)
        rq, rk, rv = _prologue_reference(qkv, h, 128, "head", blk.q_norm_weight, blk.k_norm_weight, blk.eps, rope,
                                         "interleaved")
        # text rows are normalised but not rotated
        q, k, v = dit.qkv_prologue(qkv, h, norm="head", q_weight=blk.q_norm_weight, k_weight=blk.k_norm_weight,
                                   eps=blk.eps, rope=rope)
        assert bool(((q.float() - rq).abs() <= 2.0 ** -8 * rq.abs() + 1e-6).all())
        o = torch.nn.functional.scaled_dot_product_attention(rq, rk, rv)
        ref = blk.proj(o.permute(0, 2, 1, 3).reshape(1, video + text, dim).to(torch.bfloat16)).float().detach()
        assert float((y.float() - ref).norm() / ref.norm()) < 2e-2
