"""Full multi-head GLA layer: the fp64 layer oracle against central finite differences and
closed forms (CPU), and the CUDA layer (cuBLAS projections + the library's prep / core / output kernels)
against the oracle (GPU)."""
import numpy as np
import pytest
import torch

from oracle import layer as OL


def _params(d, H, seed, dk=None, dv=None, rank=4):
    rng = np.random.default_rng(seed)
    dk = dk or d // 2
    dv = dv or d
    p = dict(W_qkvr=rng.standard_normal((d, 2 * dk + 2 * dv)) / np.sqrt(d),
             W_a1=rng.standard_normal((d, rank)) / np.sqrt(d), W_a2=rng.standard_normal((rank, dk)) / np.sqrt(rank),
             b_alpha=rng.standard_normal(dk) * 0.5, b_r=rng.standard_normal(dv) * 0.5,
             ln_w=1.0 + 0.1 * rng.standard_normal(dv), ln_b=0.1 * rng.standard_normal(dv),
             W_o=rng.standard_normal((dv, d)) / np.sqrt(dv))
    return p


NAMES = ("W_qkvr", "W_a1", "W_a2", "b_alpha", "b_r", "ln_w", "ln_b", "W_o")


def _loss(x, p, H, dy, tau):
    y, _ = OL.layer_fwd(x, *(p[n] for n in NAMES), H=H, tau=tau)
    return float((y * dy).sum())


@pytest.mark.parametrize("tau", [16.0, 1.0])
def test_layer_oracle_backward_matches_finite_differences(tau):
    """The hand-written chain rule of layer_bwd vs central differences (h = 1e-6) on every parameter and x."""
    B, T, d, H = 1, 12, 8, 2
    rng = np.random.default_rng(0)
    p = _params(d, H, 1)
    x = rng.standard_normal((B, T, d))
    dy = rng.standard_normal((B, T, d))
    y, cache = OL.layer_fwd(x, *(p[n] for n in NAMES), H=H, tau=tau)
    g = OL.layer_bwd(dy, cache, *(p[n] for n in NAMES))
    h = 1e-6
    for name in NAMES + ("x",):
        arr = x if name == "x" else p[name]
        flat = arr.reshape(-1)
        for idx in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            old = flat[idx]
            flat[idx] = old + h
            lp = _loss(x, p, H, dy, tau)
            flat[idx] = old - h
            lm = _loss(x, p, H, dy, tau)
            flat[idx] = old
            fd = (lp - lm) / (2 * h)
            got = g[name].reshape(-1)[idx]
            assert abs(got - fd) <= 1e-5 * max(1.0, abs(fd)), (name, idx, got, fd)


def test_layer_oracle_closed_forms():
    """Per-head LayerNorm output has zero mean and unit variance; with ln_w = 1, ln_b = 0 and r -> +inf
    the Swish gate passes r through, so y = (LN(O) (.) (r + b_r)) W_O exactly as the formula reads."""
    B, T, d, H = 1, 16, 8, 2
    rng = np.random.default_rng(3)
    p = _params(d, H, 2)
    x = rng.standard_normal((B, T, d))
    y, c = OL.layer_fwd(x, *(p[n] for n in NAMES), H=H)
    n = c["n"]
    np.testing.assert_allclose(n.mean(-1), 0.0, atol=1e-12)
    np.testing.assert_allclose((n ** 2).mean(-1), 1.0 - 1e-5 * c["rstd"][..., 0] ** 2, rtol=1e-9)
    p["ln_w"][:] = 1.0
    p["ln_b"][:] = 0.0
    p["b_r"][:] = 60.0                                 # sigmoid(r + 60) == 1 to fp64 precision
    y, c = OL.layer_fwd(x, *(p[n] for n in NAMES), H=H)
    dk, dv = d // 2, d
    r = (x @ p["W_qkvr"])[..., 2 * dk + dv:] + 60.0
    B_, H_, T_, V_ = c["n"].shape
    ln = c["n"].transpose(0, 2, 1, 3).reshape(B, T, dv)
    np.testing.assert_allclose(y, (ln * r) @ p["W_o"], rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("d,H,B,T", [(512, 2, 2, 192), (1024, 4, 1, 128), (2048, 4, 1, 64)])   # last: the 1.3B layer (V = 512)
def test_layer_cuda_matches_oracle(d, H, B, T):
    """GLALayer forward and every gradient against the fp64 layer oracle on the same (bf16-rounded) weights and
    inputs; bf16 tolerance 2e-2 normwise (BASELINE.json)."""
    from paper_2312_06635_b200.layer import GLALayer
    torch.manual_seed(0)
    layer = GLALayer(d, H, rank=16, device="cuda", seed=7)
    with torch.no_grad():
        layer.b_alpha.normal_(0.0, 0.5)
        layer.b_r.normal_(0.0, 0.5)
        layer.ln_w.normal_(1.0, 0.1)
        layer.ln_b.normal_(0.0, 0.1)
    gx = torch.Generator().manual_seed(11)
    x = torch.randn((B, T, d), generator=gx).bfloat16().cuda().requires_grad_(True)
    dy = torch.randn((B, T, d), generator=gx).bfloat16().cuda()
    y = layer(x)
    y.backward(dy)
    torch.cuda.synchronize()
    p = {n: getattr(layer, n).detach().double().cpu().numpy() for n in NAMES}
    xf, dyf = x.detach().double().cpu().numpy(), dy.double().cpu().numpy()
    ry, cache = OL.layer_fwd(xf, *(p[n] for n in NAMES), H=H, tau=layer.tau)
    rg = OL.layer_bwd(dyf, cache, *(p[n] for n in NAMES))

    def err(a, b):
        a = np.asarray(a, dtype=np.float64)
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
    errs = {"y": err(y.detach().float().cpu().numpy(), ry), "x": err(x.grad.float().cpu().numpy(), rg["x"])}
    for n in NAMES:
        errs[n] = err(getattr(layer, n).grad.float().cpu().numpy(), rg[n])
    # d b_alpha = sum over the B*T rows of d log alpha * sigmoid(-z) / tau, a signed sum whose terms inherit d log
    # alpha's summand-relative error (R12): its bar is relative to sum_rows |term| (reading L3).
    errs["b_alpha_strict"] = errs.pop("b_alpha")
    errs["b_alpha"] = float(np.abs(layer.b_alpha.grad.float().cpu().numpy() - rg["b_alpha"]).max() /
                            rg["b_alpha_abs"].max())
    print("layer errors vs fp64 oracle:", {k: f"{v:.2e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if not v < 2e-2 and k != "b_alpha_strict"}
    assert not bad, bad
