"""GPU parity of the upscale-aware training step (config 5) against the
reference's golden vectors: L1+SSIM loss and adjoint, the upscaled
prediction, the gradients through upscaler and rasterizer, and Adam."""

import numpy as np
import pytest

from conftest import golden, scene_of
from test_gpu_backward import FIELDS, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2503_14171_b200 as P
    return P


def test_loss_matches_reference(P):
    from paper_2503_14171_b200 import fit
    g = golden("loss")
    for lam, v, a in ((0.2, "v02", "a02"), (0.0, "v0", "a0"), (1.0, "v1", "a1")):
        value, adj = fit.loss(g["pred"], g["target"], lam)
        assert abs(value - float(g[v])) < 1e-6 * max(1.0, abs(float(g[v]))), (lam, value, float(g[v]))
        ref = g[a]
        err = np.abs(adj.double().cpu().numpy() - ref).max() / np.abs(ref).max()
        assert err < 1e-4, (lam, err)


@pytest.mark.parametrize("h,w", [(453, 200), (1080, 1920), (37, 70)])
def test_loss_matches_oracle_ragged(P, oracle, h, w):
    """The SSIM statistics walk 32-column strips in 32-row chunks over segments of tile
    rows: ragged strips, partial last chunks, several segments and a single-chunk image
    all give the oracle's value (1e-6 relative) and adjoint (1e-4 of its max, as the
    golden test: the coefficient maps and their filtering are float32)."""
    from paper_2503_14171_b200 import fit
    rng = np.random.default_rng(h * w)
    pred = rng.random((h, w, 3)).astype(np.float32)
    tgt = np.clip(pred + 0.05 * rng.standard_normal((h, w, 3)), 0, 1).astype(np.float32)
    pred[h // 3:h // 2, : w // 2] = 0.25          # flat patches: variances near the C2 floor
    tgt[h // 3:h // 2, : w // 2] = 0.25
    value, adj = fit.loss(pred, tgt, 0.2)
    rv, radj = oracle.loss(pred.astype(np.float64), tgt.astype(np.float64), 0.2)
    assert abs(value - rv) <= 1e-6 * abs(rv), (value, rv)
    assert np.abs(adj.double().cpu().numpy() - radj).max() <= 1e-4 * np.abs(radj).max()


def test_adam_groups_ragged_and_unaligned(P):
    """One launch over groups of odd sizes whose arrays start off 16-byte alignment
    (element 1 of a buffer): the vector and scalar element paths both give the
    float64 Adam update (fit.py:144-160) to rounding."""
    import torch
    from paper_2503_14171_b200 import fit
    rng = np.random.default_rng(4)
    sizes = {"a": 1, "b": 7, "c": 1030, "d": 513}
    params, grads, ref = {}, {}, {}
    for k, n in sizes.items():
        buf = torch.from_numpy(rng.normal(size=n + 1)).cuda()
        params[k] = buf[1:] if k in ("b", "d") else buf[:n]
        grads[k] = torch.from_numpy(rng.normal(size=n).astype(np.float32)).cuda()
        ref[k] = params[k].cpu().numpy().copy()
    state = fit.AdamState.like(params)
    lrs = {k: 0.01 * (i + 1) for i, k in enumerate(sizes)}
    m = {k: np.zeros(n) for k, n in sizes.items()}
    v = {k: np.zeros(n) for k, n in sizes.items()}
    for t in (1, 2):
        fit.adam_step(params, grads, state, lrs)
        for k in sizes:
            g = grads[k].double().cpu().numpy()
            m[k] = 0.9 * m[k] + 0.1 * g
            v[k] = 0.999 * v[k] + 0.001 * g * g
            ref[k] = ref[k] - lrs[k] * (m[k] / (1 - 0.9 ** t)) / (np.sqrt(v[k] / (1 - 0.999 ** t)) + 1e-8)
    for k in sizes:
        assert np.abs(params[k].cpu().numpy() - ref[k]).max() < 1e-12, k


def test_loss_validation(P):
    from paper_2503_14171_b200 import fit
    from paper_2503_14171_b200.core import DimensionError
    with pytest.raises(DimensionError):
        fit.loss(np.zeros((8, 8, 3)), np.zeros((8, 8, 3)), 0.2)     # below the SSIM window
    with pytest.raises(DimensionError):
        fit.loss(np.zeros((16, 16, 3)), np.zeros((16, 17, 3)), 0.2)


def test_training_step_matches_reference(P):
    import torch
    from paper_2503_14171_b200 import fit
    g = golden("train_step")
    sc = scene_of(g)
    tgt = torch.from_numpy(g["target"]).float().cuda()
    H, W = g["target"].shape[:2]
    lw, lh = int(g["low_w"]), int(g["low_h"])
    # the step's pieces, checked one by one
    fwd = P.render_forward(sc, lw, lh, train=True)
    pred = P.upscale_spline(fwd, 4.0, out_size=(W, H))
    assert np.abs(pred.double().cpu().numpy() - g["pred"]).max() < 1e-4
    value, adj = fit.loss_device(pred, tgt, 0.2)
    assert abs(float(value[0]) - float(g["loss"])) < 1e-5
    sadj = P.upscale_backward(fwd, 4.0, adj, out_size=(W, H))
    grads = P.render_backward(sc, fwd, P.PixelAdjoint.from_source(sadj)).numpy()
    for f in FIELDS:
        err = rel_err(grads[f], g[f])
        assert err < 1e-3, (f, err)
    # the fused trainer takes the same step; Adam vs a float64 host restatement
    tr = fit.ViewTrainer(sc, (lw, lh), (W, H), [None], [tgt], ssim_weight=0.2)
    before = {k: v.double().cpu().numpy().copy() for k, v in fit.scene_params(tr.ds).items()}
    tr.step()
    after = {k: v.double().cpu().numpy() for k, v in fit.scene_params(tr.ds).items()}
    gd = {k: v.double().cpu().numpy() for k, v in fit.grads_dict(tr.grads).items()}
    lrs = dict(fit.DEFAULT_LEARNING_RATES)
    lrs["means"] *= max(W, H)
    for k in before:
        m = 0.1 * gd[k]
        v = 0.001 * gd[k] * gd[k]
        expect = before[k] - lrs[k] * (m / 0.1) / (np.sqrt(v / 0.001) + 1e-8)
        assert np.abs(after[k] - expect).max() < 1e-10, k
    # and its gradients equal the unfused pieces' up to the float32 rounding of the
    # view-scaled rank-order terms (the trainer chains the summed terms once per step)
    for f in FIELDS:
        got, ref = tr.grads.grads().numpy()[f], grads[f]
        assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max(), f


def test_training_reduces_loss(P):
    import torch
    from paper_2503_14171_b200 import fit
    from paper_2503_14171_b200.scenes import synthetic_scene
    model = synthetic_scene(3000, 192, 108, (2.0, 6.0), seed=5)
    target_scene = synthetic_scene(3000, 192, 108, (2.0, 6.0), seed=7)
    tgt = P.render_forward(target_scene, 192, 108).color.clamp(0, 1).contiguous()
    tr = fit.ViewTrainer(model, (48, 27), (192, 108), [None], [tgt])
    first = float(tr.step()[0, 0])
    for _ in range(30):
        last = float(tr.step()[0, 0])
    assert last < first


def test_bicubic_fd_training_step_matches_oracle(P, oracle):
    """fit.py's bicubic_fd mode: FD derivative planes, their adjoint folded back (spline.py:291-297)."""
    import torch
    from paper_2503_14171_b200 import fit
    from paper_2503_14171_b200.scenes import synthetic_scene
    model = synthetic_scene(600, 96, 64, (2.0, 6.0), seed=5)
    target = np.clip(oracle.render_forward(synthetic_scene(600, 96, 64, (2.0, 6.0), seed=7), 96, 64).color, 0, 1)
    tr = fit.ViewTrainer(model, (24, 16), (96, 64), [None], [torch.from_numpy(target).float().cuda()],
                         upscale_mode="bicubic_fd")
    before = {k: v.clone() for k, v in fit.scene_params(tr.ds).items()}
    tr.step()
    got = tr.grads.grads().numpy()
    fwd = oracle.render_forward(model, 24, 16)
    src = oracle.fd_gradients(fwd.color)
    pred = oracle.upscale_spline(*src, 4.0, out_size=(96, 64))
    _, dpred = oracle.loss(pred, target, 0.2)
    sadj = oracle.upscale_backward(24, 16, 4.0, dpred, out_size=(96, 64))
    w = oracle.fd_gradients_backward(*sadj)
    z = np.zeros_like(w)
    ref = oracle.render_backward(model, fwd, (w, z, z, z))
    from test_gpu_backward import rel_err
    for f in FIELDS:
        assert rel_err(got[f], ref[f]) < 1e-3, f
    assert any(not torch.equal(before[k], v) for k, v in fit.scene_params(tr.ds).items())


def test_prefetched_targets_give_the_same_steps(P):
    """ViewTrainer.prefetch_targets (double-buffered upload on a copy stream) is
    bitwise the same training as targets resident on the device."""
    import torch
    from paper_2503_14171_b200 import fit
    from paper_2503_14171_b200.scenes import random_views, synthetic_scene
    model = synthetic_scene(3000, 96, 64, (1.0, 3.0), seed=5)
    tsc = synthetic_scene(3000, 96, 64, (1.0, 3.0), seed=7)
    views = random_views(3, 96, 64, seed=2)
    tg = [P.render_forward(tsc, 96, 64, view=v).color.clamp(0, 1).contiguous() for v in views]
    a = fit.ViewTrainer(model.copy(), (24, 16), (96, 64), views, [t.clone() for t in tg])
    b = fit.ViewTrainer(model.copy(), (24, 16), (96, 64), views, [torch.zeros_like(t) for t in tg])
    host = [t.cpu().pin_memory() for t in tg]
    for _ in range(3):
        va = a.step().clone()
        b.prefetch_targets(host)
        vb = b.step().clone()
        assert torch.equal(va, vb)
    for k in fit.scene_params(a.ds):
        assert torch.equal(fit.scene_params(a.ds)[k], fit.scene_params(b.ds)[k]), k


def test_view_parallel_step_equals_oracle_sum_of_views(P, oracle, monkeypatch):
    """Config 5's multi-GPU decomposition on one GPU: two "ranks" (trainers over views
    {0, 1} and {2, 3}) whose rank-order gradient terms are summed where the NCCL
    all-reduce sits, then chained once — equals the oracle's sum over the four views
    (1e-3 relative) and the single-rank four-view step (float32 order only)."""
    import torch
    from paper_2503_14171_b200 import fit
    from paper_2503_14171_b200.scenes import random_views, synthetic_scene, view_scene
    model = synthetic_scene(2000, 96, 64, (2.0, 6.0), seed=5)
    tsc = synthetic_scene(2000, 96, 64, (2.0, 6.0), seed=7)
    views = random_views(4, 96, 64, seed=3)
    tg = [P.render_forward(tsc, 96, 64, view=v).color.clamp(0, 1).contiguous() for v in views]
    captured = {}

    def rank1_allreduce(flat, group=None):     # rank 1's contribution to the all-reduce
        captured["b"] = flat.clone()
        return flat

    def rank0_allreduce(flat, group=None):     # rank 0 receives the SUM
        flat.add_(captured["b"])
        return flat

    b = fit.ViewTrainer(model.copy(), (24, 16), (96, 64), views[2:], tg[2:])
    monkeypatch.setattr(fit, "allreduce_grads", rank1_allreduce)
    b.step()
    a = fit.ViewTrainer(model.copy(), (24, 16), (96, 64), views[:2], tg[:2])
    monkeypatch.setattr(fit, "allreduce_grads", rank0_allreduce)
    a.step()
    monkeypatch.undo()
    full = fit.ViewTrainer(model.copy(), (24, 16), (96, 64), views, tg)
    full.step()
    got, one = a.grads.grads().numpy(), full.grads.grads().numpy()
    ref = None
    for v, t in zip(views, tg):
        sv = view_scene(model, v)
        fwd = oracle.render_forward(sv, 24, 16)
        pred = oracle.upscale_spline(fwd.color, fwd.d_dx, fwd.d_dy, fwd.d_dxdy, 4.0, out_size=(96, 64))
        _, dpred = oracle.loss(pred, t.double().cpu().numpy(), 0.2)
        sadj = oracle.upscale_backward(24, 16, 4.0, dpred, out_size=(96, 64))
        gv = oracle.render_backward(sv, fwd, sadj)
        ref = gv if ref is None else {f: ref[f] + gv[f] for f in FIELDS}
    for f in FIELDS:
        assert rel_err(got[f], ref[f]) < 1e-3, (f, rel_err(got[f], ref[f]))
        assert np.abs(got[f] - one[f]).max() <= 1e-5 * np.abs(one[f]).max(), f
