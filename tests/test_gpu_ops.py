"""K4 (CSR aggregation) and K5 (dense) parity.

F64 kernels reproduce the reference's loop order and rounding, so they are
compared bit for bit with the compiled reference (oracle/_ref) / golden
vectors; F32 kernels are compared with a float64 numpy reference of the same
op at the stated tolerance (rtol 1e-5 on O(1) values)."""
import os

import numpy as np
import pytest
import torch

from oracle import port
from paper_2306_01381_b200 import ops

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _view_from_golden():
    """Rebuild device arrays of the reference DeviceAggView of device 1 (owner p4/s11)."""
    from oracle.oracle import RefView  # noqa: F401  (import only for the type)
    import oracle
    if oracle.ref_available():
        return oracle.ref.view(G["g_adj_ptr"], G["g_adj"], G["g_owner_p4_s11"], 4, 1).v
    pytest.skip("compiled reference not present")


def _t(a, dt=None):
    a = np.ascontiguousarray(a)
    t = torch.as_tensor(a, device="cuda")
    return t if dt is None else t.to(dt)


def test_aggregate_rows_f64_bit_exact(cuda):
    v = _view_from_golden()
    h, hr = G["agg_h"], G["agg_hr"]
    out = torch.zeros(h.shape, dtype=torch.float64, device=cuda)
    ops.csr_aggregate(_t(h), _t(v["local_ptr"]), _t(v["local_row"]), _t(v["local_alpha_fwd"]),
                      out, self_alpha=_t(v["self_alpha"]), y=_t(hr), ptr_b=_t(v["remote_ptr"]),
                      col_b=_t(v["remote_slot"]), alpha_b=_t(v["remote_alpha"]))
    assert (out.cpu().numpy() == G["agg_out"]).all()
    # row subset: central rows only, others untouched (aggregate.hpp:92-93)
    out2 = torch.full(h.shape, 7.0, dtype=torch.float64, device=cuda)
    rows = _t(v["central"].astype(np.int32))
    ops.csr_aggregate(_t(h), _t(v["local_ptr"]), _t(v["local_row"]), _t(v["local_alpha_fwd"]),
                      out2, self_alpha=_t(v["self_alpha"]), y=_t(hr), ptr_b=_t(v["remote_ptr"]),
                      col_b=_t(v["remote_slot"]), alpha_b=_t(v["remote_alpha"]), rows=rows)
    o2 = out2.cpu().numpy()
    c = v["central"]
    assert (o2[c] == G["agg_out"][c]).all()
    mask = np.ones(len(o2), bool)
    mask[c] = False
    assert (o2[mask] == 7.0).all()


def test_backward_local_and_partials_f64_bit_exact(cuda):
    v = _view_from_golden()
    gb = G["agg_gbar"]
    out = torch.zeros(gb.shape, dtype=torch.float64, device=cuda)
    ops.csr_aggregate(_t(gb), _t(v["local_ptr"]), _t(v["local_row"]), _t(v["local_alpha_bwd"]),
                      out, self_alpha=_t(v["self_alpha"]))
    assert (out.cpu().numpy() == G["agg_bwd_local"]).all()
    # partials through the transposed remote CSR (slot -> marginal rows ascending)
    nr = len(v["slot_node"])
    rp, rs_, ra = v["remote_ptr"], v["remote_slot"], v["remote_alpha"]
    lists = [[] for _ in range(nr)]
    for r in v["marginal"]:
        for e in range(rp[r], rp[r + 1]):
            lists[rs_[e]].append((r, ra[e]))
    sp = np.zeros(nr + 1, np.int64)
    sp[1:] = np.cumsum([len(x) for x in lists])
    srow = np.array([r for x in lists for r, _ in x], np.int32)
    sal = np.array([a for x in lists for _, a in x])
    part = torch.zeros((nr, gb.shape[1]), dtype=torch.float64, device=cuda)
    ops.csr_aggregate(_t(gb), _t(sp), _t(srow), _t(sal), part)
    assert (part.cpu().numpy() == G["agg_partials"]).all()


@pytest.mark.parametrize("d", [100, 256, 602, 37])
def test_aggregate_f32_tolerance(cuda, d):
    rs = np.random.default_rng(d)
    n, nh, deg = 3000, 500, 20
    ptr = np.arange(0, (n + 1) * deg, deg, dtype=np.int64)
    col = rs.integers(0, n, n * deg).astype(np.int32)
    al = rs.uniform(0, 0.2, n * deg)
    rptr = np.arange(0, (n + 1) * 3, 3, dtype=np.int64)
    rcol = rs.integers(0, nh, n * 3).astype(np.int32)
    ral = rs.uniform(0, 0.2, n * 3)
    sa = rs.uniform(0, 1, n)
    h = rs.standard_normal((n, d))
    hr = rs.standard_normal((nh, d))
    exp = sa[:, None] * h
    for r in range(n):
        exp[r] += (al[ptr[r]:ptr[r + 1], None] * h[col[ptr[r]:ptr[r + 1]]]).sum(0)
        exp[r] += (ral[rptr[r]:rptr[r + 1], None] * hr[rcol[rptr[r]:rptr[r + 1]]]).sum(0)
    f = torch.float32
    out = torch.zeros((n, d), dtype=f, device=cuda)
    ops.csr_aggregate(_t(h, f), _t(ptr), _t(col), _t(al, f), out, self_alpha=_t(sa, f),
                      y=_t(hr, f), ptr_b=_t(rptr), col_b=_t(rcol), alpha_b=_t(ral, f))
    assert np.allclose(out.cpu().numpy(), exp, rtol=1e-5, atol=1e-5)


def test_dense_f64_bit_exact(cuda):
    h, w0, dz = G["agg_h"], G["w0"], G["dense_dz"]
    n = h.shape[0]
    out = torch.zeros((n, 12), dtype=torch.float64, device=cuda)
    ops.dense_forward(_t(h), _t(w0), out, relu=True)
    assert (out.cpu().numpy() == G["dense_fwd"]).all()
    ig = torch.zeros((n, 8), dtype=torch.float64, device=cuda)
    ops.dense_input_grad(_t(dz), _t(w0), ig)
    assert (ig.cpu().numpy() == G["dense_igrad"]).all()
    wg = torch.zeros((8, 12), dtype=torch.float64, device=cuda)
    ops.dense_weight_grad(_t(h), _t(dz), wg)
    assert (wg.cpu().numpy() == G["dense_wgrad"]).all()


@pytest.mark.parametrize("din,dout", [(100, 256), (256, 256), (256, 47), (602, 256)])
def test_dense_f32_against_fp64(cuda, din, dout):
    rs = np.random.default_rng(din * 1000 + dout)
    n = 5000
    a = rs.standard_normal((n, din))
    w = rs.standard_normal((din, dout)) / np.sqrt(din)
    f = torch.float32
    z = a @ w
    out = torch.zeros((n, dout), dtype=f, device=cuda)
    ops.dense_forward(_t(a, f), _t(w, f), out, relu=True)
    assert np.allclose(out.cpu().numpy(), np.maximum(z, 0), rtol=1e-4, atol=1e-4)
    dz = rs.standard_normal((n, dout))
    ig = torch.zeros((n, din), dtype=f, device=cuda)
    ops.dense_input_grad(_t(dz, f), _t(w, f), ig)
    assert np.allclose(ig.cpu().numpy(), dz @ w.T, rtol=1e-4, atol=1e-4)
    wg = torch.ones((din, dout), dtype=f, device=cuda)
    ops.dense_weight_grad(_t(a, f), _t(dz, f), wg, accumulate=True)
    ref = 1.0 + a.T @ dz
    assert np.allclose(wg.cpu().numpy(), ref, rtol=1e-4, atol=1e-3 * np.sqrt(n) * 1e-2)
    # deterministic: identical bits on repeat
    wg2 = torch.ones((din, dout), dtype=f, device=cuda)
    ops.dense_weight_grad(_t(a, f), _t(dz, f), wg2, accumulate=True)
    assert torch.equal(wg, wg2)


@pytest.mark.parametrize("n", [129, 300, 5121, 33000])
@pytest.mark.parametrize("din,dout", [(100, 256), (256, 256), (256, 47), (47, 256)])
def test_dense_f32_tile_edges(cuda, n, din, dout):
    """Row counts around the tile grid: odd tile counts (the 2-CTA cluster path pads
    the row tiles to a multiple of 2: the padding tile is TMA zero fill and must
    not be stored), single tiles (no cluster), 256-row tiles for narrow outputs."""
    rs = np.random.default_rng(n + din * 7 + dout)
    a = rs.standard_normal((n, din))
    w = rs.standard_normal((din, dout)) / np.sqrt(din)
    f = torch.float32
    out = torch.full((n + 200, dout), -3.0, dtype=f, device=cuda)
    ops.dense_forward(_t(a, f), _t(w, f), out[:n], relu=True)
    o = out.cpu().numpy()
    assert np.allclose(o[:n], np.maximum(a @ w, 0), rtol=1e-4, atol=1e-4)
    assert (o[n:] == -3.0).all()
    ig = torch.full((n + 200, din), -3.0, dtype=f, device=cuda)
    dz = rs.standard_normal((n, dout))
    ops.dense_input_grad(_t(dz, f), _t(w, f), ig[:n])
    g = ig.cpu().numpy()
    assert np.allclose(g[:n], dz @ w.T, rtol=1e-4, atol=1e-4)
    assert (g[n:] == -3.0).all()


@pytest.mark.parametrize("din,dout", [(602, 300), (300, 602), (128, 512)])
def test_dense_f32_wide_outputs(cuda, din, dout):
    """Outputs wider than one TMEM tile (N > 256: 602-wide input gradients of the
    Reddit-shaped first layer, hidden 512) run on the tcgen05 path as 256-column
    blocks of B: same tolerance as the single-block shapes."""
    rs = np.random.default_rng(din * 7 + dout)
    n = 3000
    a = rs.standard_normal((n, din))
    w = rs.standard_normal((din, dout)) / np.sqrt(din)
    f = torch.float32
    out = torch.zeros((n, dout), dtype=f, device=cuda)
    ops.dense_forward(_t(a, f), _t(w, f), out, relu=True)
    assert np.allclose(out.cpu().numpy(), np.maximum(a @ w, 0), rtol=1e-4, atol=1e-4)
    dz = rs.standard_normal((n, dout))
    ig = torch.zeros((n, din), dtype=f, device=cuda)
    ops.dense_input_grad(_t(dz, f), _t(w, f), ig)
    assert np.allclose(ig.cpu().numpy(), dz @ w.T, rtol=1e-4, atol=1e-4)


def test_dense_row_subsets(cuda):
    rs = np.random.default_rng(3)
    n, din, dout = 1000, 64, 48
    a = rs.standard_normal((n, din)).astype(np.float32)
    w = rs.standard_normal((din, dout)).astype(np.float32)
    rows = np.sort(rs.choice(n, 300, replace=False)).astype(np.int32)
    out = torch.full((n, dout), -3.0, device=cuda)
    ops.dense_forward(_t(a), _t(w), out, relu=False, rows=_t(rows))
    o = out.cpu().numpy()
    assert np.allclose(o[rows], a[rows] @ w, rtol=1e-4, atol=1e-4)
    m = np.ones(n, bool)
    m[rows] = False
    assert (o[m] == -3.0).all()
    out2 = torch.zeros((n, dout), device=cuda)
    ops.dense_forward(_t(a), _t(w), out2, relu=True, row_begin=100, n_rows=50)
    assert np.allclose(out2.cpu().numpy()[100:150], np.maximum(a[100:150] @ w, 0), atol=1e-4)
    wg = torch.zeros((din, dout), device=cuda)
    ops.dense_weight_grad(_t(a), _t(a[:, :dout].copy()), wg, rows=_t(rows))
    assert np.allclose(wg.cpu().numpy(), a[rows].T @ a[rows, :dout], rtol=1e-4, atol=1e-3)


def test_loss_adam_relu(cuda):
    rs = np.random.default_rng(9)
    n, c = 500, 7
    logits = rs.standard_normal((n, c))
    labels = rs.integers(0, c, n).astype(np.int32)
    rows = np.sort(rs.choice(n, 200, replace=False)).astype(np.int32)
    grad = torch.zeros((n, c), dtype=torch.float64, device=cuda)
    loss = ops.masked_ce(_t(logits), _t(labels), _t(rows), 1 / 300, grad)
    el, eg = port.masked_ce_partial(logits, labels, rows, 1 / 300)
    assert abs(loss - el) < 1e-12 * max(1, abs(el))
    assert np.allclose(grad.cpu().numpy(), eg, rtol=1e-12, atol=1e-15)
    hits = ops.count_correct(_t(logits), _t(labels), _t(rows))
    assert hits == int((logits[rows].argmax(1) == labels[rows]).sum())
    p = rs.standard_normal(1000)
    m, v = np.zeros(1000), np.zeros(1000)
    gr = rs.standard_normal(1000)
    pt, mt, vt = _t(p), _t(m), _t(v)
    for t in (1, 2, 3):
        ops.adam_step(pt, mt, vt, _t(gr), t)
        port.adam_step(p, m, v, gr, t)
    assert (pt.cpu().numpy() == p).all()  # f64 Adam is bit-exact (optim.hpp:47-62)
    act = rs.standard_normal((50, 9))
    act[act < 0] = 0
    dh = rs.standard_normal((50, 9))
    dz = torch.zeros((50, 9), dtype=torch.float64, device=cuda)
    ops.relu_backward(_t(act), _t(dh), dz)
    assert (dz.cpu().numpy() == np.where(act <= 0, 0, dh)).all()
