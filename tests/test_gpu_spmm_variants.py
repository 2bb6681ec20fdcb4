"""Every production fp32 K4 variant against the oracle (aggregate.hpp:94-165).

The engine's SpMM dispatch (spmm.cu:spmm_f32, through the C-ABI
qgnn_spmm_plan_*) is checked directly against the C restatement of
aggregate_rows (oracle/qgnn_oracle.c:qo_aggregate_rows, fp64) on a power-law
graph with hub rows, a remote (halo) CSR and the ReLU-backward mask, for every
width class and every run-time variant switch:

* <= 64 wide: k_spmm_sorted (12- and 16-register builds), rows degree-sorted,
  hub segments finished in-kernel by arrival counters or by k_spmm_hubred;
* <= 128 wide: k_spmm_f32g2 (hub segments merged / separate) and k_spmm_f32g;
* 256 wide: k_spmm_wide (32- and 16-byte gathers), k_spmm_wide_half
  (half-warp rows), k_spmm_f32<2>;
* other widths (300, 602): k_spmm_f32<NV>.

Tolerance: fp32 FMA accumulation vs fp64 — |gpu - oracle| <= 1e-5 * sum|alpha x|
+ 1e-6 per element (the row's absolute-sum scale).
"""
import numpy as np
import pytest
import torch

from oracle import port
from paper_2306_01381_b200 import ops
from synth import generate_planted

pytestmark = pytest.mark.gpu

N_HALO = 3000


@pytest.fixture(scope="module")
def graph():
    g = generate_planted(6000, 60000, 8, 4, 1, 0.0, gamma=2.1, seed=5)
    ptr, adj = g["adj_ptr"], g["adj"]
    n = len(ptr) - 1
    rs = np.random.default_rng(1)
    deg = np.diff(ptr)
    assert deg.max() > 300  # hub rows exist at the default threshold too
    alpha = rs.uniform(-1, 1, len(adj))
    sa = rs.uniform(-1, 1, n)
    # remote CSR over a halo table: a few remote neighbours per row, some heavy rows
    rdeg = rs.poisson(2.0, n)
    rdeg[rs.choice(n, 20, replace=False)] = rs.integers(150, 600, 20)
    rptr = np.concatenate([[0], np.cumsum(rdeg)]).astype(np.int64)
    rslot = rs.integers(0, N_HALO, int(rptr[-1])).astype(np.int32)
    ralpha = rs.uniform(-1, 1, len(rslot))
    return dict(n=n, ptr=ptr, adj=adj, alpha=alpha, sa=sa, rptr=rptr, rslot=rslot,
                ralpha=ralpha)


def _dev(a, dt=None):
    return torch.as_tensor(np.ascontiguousarray(a if dt is None else a.astype(dt)), device="cuda")


def _padded(rs, rows, dim, relu_like=False):
    ld = -(-dim // 8) * 8
    x = np.zeros((rows, ld), np.float32)
    v = rs.standard_normal((rows, dim)).astype(np.float32)
    if relu_like:
        v[v < 0.3] = 0.0
    x[:, :dim] = v
    return x


def _check(g, dim, remote, mask, hub_deg, row_range=None):
    rs = np.random.default_rng(dim * 7 + hub_deg + remote * 3 + mask * 5)
    n = g["n"]
    r0, r1 = row_range or (0, n)
    x = _padded(rs, n, dim)
    y = _padded(rs, N_HALO, dim) if remote else None
    m = _padded(rs, n, dim, relu_like=True) if mask else None
    # oracle in fp64 on the same fp32 inputs (alphas rounded to fp32 as the GPU sees them)
    a32 = g["alpha"].astype(np.float32).astype(np.float64)
    ra32 = g["ralpha"].astype(np.float32).astype(np.float64)
    sa32 = g["sa"].astype(np.float32).astype(np.float64)
    v = dict(self_alpha=sa32, local_ptr=g["ptr"], local_row=g["adj"], local_alpha_fwd=a32,
             remote_ptr=g["rptr"] if remote else None, remote_slot=g["rslot"] if remote else None,
             remote_alpha=ra32 if remote else None)
    rows = np.arange(r0, r1, dtype=np.int32)
    exp = np.zeros((n, dim))
    port.aggregate_rows(v, x[:, :dim].astype(np.float64),
                        y[:, :dim].astype(np.float64) if remote else None, rows, exp)
    # scale: sum of |terms| per element
    ax = np.abs(x[:, :dim]).astype(np.float64)
    scale = np.zeros((n, dim))
    va = dict(v, self_alpha=np.abs(sa32), local_alpha_fwd=np.abs(a32),
              remote_alpha=np.abs(ra32) if remote else None)
    port.aggregate_rows(va, ax, np.abs(y[:, :dim]).astype(np.float64) if remote else None, rows,
                        scale)
    if mask:
        exp = np.where(m[:, :dim] > 0, exp, 0.0)
    plan = ops.SpmmPlan(g["ptr"], r0, r1 - r0, dim, ptr_b=g["rptr"] if remote else None,
                        hub_deg=hub_deg)
    out = torch.full((n, x.shape[1]), 7.0, dtype=torch.float32, device="cuda")
    plan.run(dim, _dev(x), _dev(g["ptr"]), _dev(g["adj"]), _dev(g["alpha"], np.float32), out,
             self_alpha=_dev(g["sa"], np.float32), y=_dev(y) if remote else None,
             ptr_b=_dev(g["rptr"]) if remote else None, col_b=_dev(g["rslot"]) if remote else None,
             alpha_b=_dev(g["ralpha"], np.float32) if remote else None,
             mask=_dev(m) if mask else None)
    ops.sync_check()
    got = out.cpu().numpy()
    err = np.abs(got[r0:r1, :dim] - exp[r0:r1])
    tol = 1e-5 * scale[r0:r1] + 1e-6
    bad = np.argwhere(err > tol)
    assert len(bad) == 0, (dim, remote, mask, hub_deg, bad[:5], err.max())
    # rows outside the range are untouched
    if r0 > 0:
        assert (got[:r0] == 7.0).all()
    if r1 < n:
        assert (got[r1:] == 7.0).all()
    # a second run reuses the hub arrival counters (reset in-kernel): same bits
    out2 = torch.full_like(out, 7.0)
    plan.run(dim, _dev(x), _dev(g["ptr"]), _dev(g["adj"]), _dev(g["alpha"], np.float32), out2,
             self_alpha=_dev(g["sa"], np.float32), y=_dev(y) if remote else None,
             ptr_b=_dev(g["rptr"]) if remote else None, col_b=_dev(g["rslot"]) if remote else None,
             alpha_b=_dev(g["ralpha"], np.float32) if remote else None,
             mask=_dev(m) if mask else None)
    assert torch.equal(out, out2)
    plan.close()


DIMS = [40, 47, 48, 64, 100, 128, 256, 300, 602]


@pytest.mark.parametrize("dim", DIMS)
@pytest.mark.parametrize("remote", [False, True])
@pytest.mark.parametrize("hub_deg", [128, 2])
def test_spmm_default_dispatch(cuda, graph, dim, remote, hub_deg):
    _check(graph, dim, remote, mask=False, hub_deg=hub_deg)


@pytest.mark.parametrize("dim", [47, 100, 256])
@pytest.mark.parametrize("remote", [False, True])
def test_spmm_relu_mask_epilogue(cuda, graph, dim, remote):
    _check(graph, dim, remote, mask=True, hub_deg=128)
    _check(graph, dim, remote, mask=True, hub_deg=2)


def test_spmm_row_subrange(cuda, graph):
    n = graph["n"]
    for dim in (48, 100, 256):
        _check(graph, dim, True, mask=False, hub_deg=64, row_range=(n // 3, 2 * n // 3 + 7))


# run-time switches: each selects another kernel for the same call
SWITCHES = [
    ({"QGNN_SPMM_SORTED": "0"}, [40, 47, 64]),            # narrow rows via k_spmm_f32g2
    ({"QGNN_SPMM_SORTED": "2"}, [40, 47, 64]),            # 16-register sorted build
    ({"QGNN_HUB_FINISH": "0"}, [47, 100, 256]),           # separate k_spmm_hubred
    ({"QGNN_HUB_MERGE": "0"}, [100, 256]),                # separate k_spmm_hubseg launch
    ({"QGNN_SPMM_HALF_DEG": "1000"}, [256]),              # k_spmm_wide_half
    ({"QGNN_SPMM_HALF_DEG": "1000", "QGNN_HUB_FINISH": "0"}, [256]),
    ({"QGNN_SPMM_LD256": "0"}, [47, 100, 256]),           # 16-byte gathers
    ({"QGNN_SPMM_WIDE": "0"}, [256]),                     # k_spmm_f32<2>
    ({"QGNN_SPMM_G2": "0"}, [100, 128]),                  # k_spmm_f32g
    ({"QGNN_SPMM_GROUPED": "0"}, [100, 128]),             # k_spmm_f32<1>
    ({"QGNN_G2_MINB": "3"}, [100]),
]


@pytest.mark.parametrize("env,dims", SWITCHES, ids=[",".join(f"{k}={v}" for k, v in e.items())
                                                    for e, _ in SWITCHES])
def test_spmm_variant_switches(cuda, graph, monkeypatch, env, dims):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for dim in dims:
        for remote in (False, True):
            for hub_deg in (128, 2):
                _check(graph, dim, remote, mask=remote, hub_deg=hub_deg)
