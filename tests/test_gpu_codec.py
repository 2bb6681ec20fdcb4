"""K1/K3 parity: GPU quantize+pack and unpack+dequantize vs the oracle and the
reference's golden vectors.  Integer/byte outputs must be bit-exact."""
import os

import numpy as np
import pytest
import torch

from oracle import port
from paper_2306_01381_b200 import DecodeError, InvalidArgument, WIRE_GPU, WIRE_REF, ops

pytestmark = pytest.mark.gpu
GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
DIMS = [100, 128, 200, 256, 300, 602]


def _gpu_quantize_one(h, b, key, layout, dtype=torch.float64):
    v = torch.as_tensor(np.asarray(h)[None, :], dtype=dtype, device="cuda")
    wire, idx = ops.encode_message_set(v, [0], [0], [b], ops.lib.qgnn_rng_fork(key, 0) if False
                                       else key, layout=layout)
    return wire.cpu().numpy(), idx


def test_encode_golden_byte_identical(cuda):
    G = GOLDEN
    c = [int(x) for x in G["enc_coords"]]
    key = port.stream(c[0], *c[1:])
    vals = torch.as_tensor(G["enc_vals"], device=cuda)
    wire, idx = ops.encode_message_set(vals, G["enc_rows"], G["enc_ids"], G["enc_bits"], key,
                                       layout=WIRE_REF)
    assert wire.cpu().numpy().tobytes() == G["enc_wire"].tobytes()
    assert (G["enc_ids"][idx["pos"]] == G["enc_idx_id"]).all()
    dec = ops.decode_message_set(wire, idx["bits"], idx["off"], 96, dtype=torch.float64,
                                 layout=WIRE_REF)
    assert (dec.cpu().numpy() == G["enc_decoded"]).all()


def test_quantize_golden_vectors(cuda):
    """Every reference golden row (dims 1..602, b 2/4/8, gauss/relu/const)."""
    for i in range(int(GOLDEN["n_quant"])):
        meta = GOLDEN[f"q{i}_meta"].astype(np.uint64)
        b, seed, coords = int(meta[0]), int(meta[1]), [int(x) for x in meta[2:]]
        h = GOLDEN[f"q{i}_h"]
        # message key = fork(set_key, id): use set = stream(seed, coords[:-1]), id = coords[-1]
        set_key = port.stream(seed, *coords[:-1])
        v = torch.as_tensor(h[None, :], device=cuda)
        wire, idx = ops.encode_message_set(v, [0], [coords[-1]], [b], set_key, layout=WIRE_REF)
        w = wire.cpu().numpy()
        assert w[0] == b
        s = w[9:17].view(np.float64)[0]
        z = w[17:25].view(np.float64)[0]
        es, ez = GOLDEN[f"q{i}_sz"]
        assert s == es and z == ez, i
        assert (w[25:] == GOLDEN[f"q{i}_payload"]).all(), i


def _random_rows(rs, n, d, kind):
    x = rs.standard_normal((n, d)) * rs.uniform(0.05, 5.0, (n, 1))
    if kind == "relu":
        x = np.maximum(x, 0.0)
        x[:: 17] = 0.0  # all-zero rows -> S = 0 path
    elif kind == "const":
        x[:] = rs.standard_normal((n, 1))
    return x


@pytest.mark.parametrize("d", DIMS)
def test_random_sets_f64_reference_layout_bit_exact(cuda, d):
    rs = np.random.default_rng(d)
    for kind in ("gauss", "relu", "const"):
        n = 257
        x = _random_rows(rs, n, d, kind)
        rows = rs.permutation(n)[:200]
        ids = (rs.permutation(100000)[:200] * 3 + 1).astype(np.uint32)
        bits = rs.choice([2, 4, 8], 200).astype(np.int32)
        key = port.stream(7, 2, 3, 1, 0, 2)
        exp_wire, pos, off = port.encode_message_set(x, rows, ids, bits, key)
        wire, idx = ops.encode_message_set(torch.as_tensor(x, device=cuda), rows, ids, bits, key,
                                           layout=WIRE_REF)
        assert wire.cpu().numpy().tobytes() == exp_wire.tobytes()
        dec = ops.decode_message_set(wire, idx["bits"], idx["off"], d, dtype=torch.float64,
                                     layout=WIRE_REF)
        exp = port.decode_message_set(exp_wire, bits[pos], np.full(200, d, np.uint64), off,
                                      len(exp_wire))
        assert (dec.cpu().numpy() == exp).all()


@pytest.mark.parametrize("d", DIMS)
def test_random_sets_f32_gpu_layout(cuda, d):
    """fp32 buffers: codes bit-exact with the oracle fed the same fp32 values as
    doubles; headers are (float)S, (float)Z; dequant within fp32 rounding."""
    rs = np.random.default_rng(1000 + d)
    for kind in ("gauss", "relu"):
        n = 300
        x32 = _random_rows(rs, n, d, kind).astype(np.float32)
        x = x32.astype(np.float64)
        rows = np.arange(n)
        ids = np.arange(n, dtype=np.uint32) * 5
        bits = rs.choice([2, 4, 8], n).astype(np.int32)
        key = port.stream(3, 2, 1, 0, 0, 1)
        wire, idx = ops.encode_message_set(torch.as_tensor(x32, device=cuda), rows, ids, bits,
                                           key, layout=WIRE_GPU)
        w = wire.cpu().numpy()
        for k in range(n):
            i = idx["pos"][k]
            o = int(idx["off"][k])
            b = int(bits[i])
            s, z, p = port.quantize(x[rows[i]], b, port.fork(key, int(ids[i])))
            hdr = w[o:o + 16]
            assert hdr[:4].view(np.float32)[0] == np.float32(s)
            assert hdr[4:8].view(np.float32)[0] == np.float32(z)
            assert hdr[8:12].view(np.uint32)[0] == d and hdr[12] == b
            nb = len(p)
            assert (w[o + 16:o + 16 + nb] == p).all(), (k, b)
            assert (w[o + 16 + nb:o + 16 + ((nb + 15) // 16) * 16] == 0).all()
        dec = ops.decode_message_set(wire, idx["bits"], idx["off"], d, dtype=torch.float32)
        got = dec.cpu().numpy().astype(np.float64)
        for k in range(0, n, 7):
            i = idx["pos"][k]
            b = int(bits[i])
            s, z, p = port.quantize(x[rows[i]], b, port.fork(key, int(ids[i])))
            exp = port.dequantize(p, b, d, s, z)
            assert np.allclose(got[k], exp, rtol=2e-6, atol=2e-6 * (abs(s) * 255 + abs(z)))


def test_scatter_and_accumulate(cuda):
    rs = np.random.default_rng(4)
    d, n = 64, 100
    x = rs.standard_normal((n, d)).astype(np.float32)
    bits = np.full(n, 8, np.int32)
    wire, idx = ops.encode_message_set(torch.as_tensor(x, device=cuda), np.arange(n),
                                       np.arange(n), bits, 123)
    out = torch.ones((2 * n, d), dtype=torch.float32, device=cuda)
    dst = torch.as_tensor((np.arange(n) * 2 + 1).astype(np.int32), device=cuda)
    b_t = torch.as_tensor(idx["bits"].astype(np.uint8), device=cuda)
    o_t = torch.as_tensor(idx["off"].view(np.int64), device=cuda)
    ops.dequant_scatter(wire, b_t, o_t, d, out, dst_rows=dst, accumulate=True)
    o = out.cpu().numpy()
    assert (o[0::2] == 1).all()
    dec = ops.decode_message_set(wire, idx["bits"], idx["off"], d).cpu().numpy()
    assert np.allclose(o[1::2], dec + 1, atol=1e-6)
    step = (x.max(1) - x.min(1)) / 255
    assert (np.abs(dec - x) <= step[:, None] * 1.0001 + 1e-6).all()  # within one step


def test_nonfinite_input_raises_invalid_argument(cuda):
    x = torch.zeros((2, 16), dtype=torch.float32, device=cuda)
    x[1, 3] = float("nan")
    with pytest.raises(InvalidArgument):
        ops.encode_message_set(x, [0, 1], [0, 1], [4, 4], 5)
    ops.encode_message_set(x, [0], [0], [4], 5)  # error word was cleared


def test_corrupt_chunk_raises_decode_error(cuda):
    x = torch.randn((3, 16), device=cuda)
    wire, idx = ops.encode_message_set(x, [0, 1, 2], [0, 1, 2], [4, 4, 8], 5)
    with pytest.raises(DecodeError):
        ops.decode_message_set(wire, np.array([4, 8, 8]), idx["off"], 16)
    bad = wire.clone()
    bad[int(idx["off"][0]) + 8] = 15  # count field
    with pytest.raises(DecodeError):
        ops.decode_message_set(bad, idx["bits"], idx["off"], 16)


def test_unbiased_at_scale(cuda):
    """Size-independent property at a large size: E[dequant] = x within 4 SE."""
    rs = np.random.default_rng(8)
    d, n = 256, 20000
    base = rs.standard_normal(d).astype(np.float32)
    x = np.tile(base, (n, 1))
    for b in (2, 8):
        wire, idx = ops.encode_message_set(torch.as_tensor(x, device=cuda), np.arange(n),
                                           np.arange(n), np.full(n, b), 77)
        dec = ops.decode_message_set(wire, idx["bits"], idx["off"], d).cpu().numpy()
        s = (base.max() - base.min()) / ((1 << b) - 1)
        mean = dec.astype(np.float64).mean(0)  # fp32 axis-0 means accumulate naively
        se = s / 2 / np.sqrt(n)
        assert (np.abs(mean - base) < 4 * se + 1e-6).mean() > 0.99


def test_fast_path_codes_exact_on_adversarial_rows(cuda):
    """K1's reciprocal fast path must reproduce the exact-division codes: lattice
    rows (x exactly integral), near-lattice rows, constant and post-ReLU rows."""
    rs = np.random.default_rng(77)
    rows = []
    for k in range(3000):
        b = (2, 4, 8)[k % 3]
        lv = (1 << b) - 1
        kind = k % 6
        if kind == 0:
            x = rs.standard_normal(256)
        elif kind == 1:  # exact lattice: (h - lo) / S integral
            x = rs.integers(0, lv + 1, 256).astype(np.float64) * 0.375 - 1.5
        elif kind == 2:  # lattice plus one-ulp-scale noise
            x = rs.integers(0, lv + 1, 256) * 0.25 + rs.standard_normal(256) * 1e-7
        elif kind == 3:
            x = np.maximum(rs.standard_normal(256), 0)
        elif kind == 4:
            x = rs.standard_normal(256) * 1e-30
        else:
            x = rs.uniform(-1e4, 1e4, 256)
        rows.append((x.astype(np.float32), b))
    X = np.stack([r[0] for r in rows])
    bits = np.array([r[1] for r in rows], np.int32)
    n = len(rows)
    ids = np.arange(n, dtype=np.uint32) * 7 + 1
    key = port.stream(9, 2, 4, 1, 2, 3)
    wire, idx = ops.encode_message_set(torch.as_tensor(X, device=cuda), np.arange(n), ids, bits,
                                       key, layout=WIRE_GPU)
    w = wire.cpu().numpy()
    bad = 0
    for k in range(n):
        i = idx["pos"][k]
        o = int(idx["off"][k])
        s_, z_, p = port.quantize(X[i].astype(np.float64), int(bits[i]), port.fork(key, int(ids[i])))
        bad += int(not (w[o + 16:o + 16 + len(p)] == p).all())
    assert bad == 0


K1_DIMS = [3, 4, 5, 12, 13, 16, 20, 36, 47, 64, 68, 100, 101, 128, 256, 260, 500, 512, 516, 602,
           1000, 1024]


def _k1_rows(rs, kind, n, d, lv):
    if kind == "gauss":
        return rs.standard_normal((n, d))
    if kind == "negzero":  # post-ReLU rows holding -0.0: first-occurrence signed zero
        x = np.maximum(rs.standard_normal((n, d)), 0.0)
        x[rs.random((n, d)) < 0.2] = -0.0
        x[::5] = -0.0
        x[1::5, 0] = 0.0
        return x
    if kind == "lattice":  # x = (h - lo) / S exactly integral, and one-ulp-scale noise
        x = rs.integers(0, lv + 1, (n, d)) * 0.375 - 1.5
        x[1::2] += rs.standard_normal((n // 2, d)) * 1e-7
        return x
    if kind == "tiny":
        return rs.standard_normal((n, d)) * 1e-30
    if kind == "huge":  # S > 2^100: the fp32 decision is off, every element exact
        return rs.standard_normal((n, d)) * 1e36
    x = np.repeat(rs.standard_normal((n, 1)), d, 1)  # constant rows: S = 0, no draws
    x[::2, rs.integers(0, d)] += 1.0
    return x


@pytest.mark.parametrize("d", K1_DIMS)
def test_k1_grouped_kernel_bit_exact(cuda, d):
    """Production K1 (grouped lanes, fp32 decision with exact fallback) at every
    lane-group shape: codes, headers and zero padding equal the oracle's."""
    rs = np.random.default_rng(5000 + d)
    ld = (d + 7) // 8 * 8
    for kind in ("gauss", "negzero", "lattice", "tiny", "huge", "const"):
        n = 48
        bits = np.array([(2, 4, 8)[k % 3] for k in range(n)], np.int32)
        x32 = np.zeros((n, ld), np.float32)
        for b in (2, 4, 8):
            sel = bits == b
            x32[sel, :d] = _k1_rows(rs, kind, int(sel.sum()), d, (1 << b) - 1)
        x32[:, d:] = np.nan  # row padding is never read as data
        xt = torch.as_tensor(x32, device=cuda)[:, :d]
        ids = (rs.permutation(50000)[:n] * 2 + 1).astype(np.uint32)
        key = port.stream(11, 2, 3, 0, 1, 2)
        wire, idx = ops.encode_message_set(xt, np.arange(n), ids, bits, key, layout=WIRE_GPU)
        w = wire.cpu().numpy()
        for k in range(n):
            i = idx["pos"][k]
            o = int(idx["off"][k])
            b = int(bits[i])
            s, z, p = port.quantize(x32[i, :d].astype(np.float64), b, port.fork(key, int(ids[i])))
            hdr = w[o:o + 16]
            assert hdr[:4].view(np.float32)[0] == np.float32(s), (kind, k)
            assert hdr[4:8].view(np.float32)[0] == np.float32(z), (kind, k)
            assert hdr[8:12].view(np.uint32)[0] == d and hdr[12] == b
            nb = len(p)
            assert (w[o + 16:o + 16 + nb] == p).all(), (kind, k, b)
            assert (w[o + 16 + nb:o + 16 + ((nb + 15) // 16) * 16] == 0).all(), (kind, k, b)


def test_k1_production_matches_round1_kernel_at_scale(cuda):
    """400k messages per (dim, width): the grouped K1 writes the same wire bytes
    as the round-1 lean kernel (itself bit-exact against the oracle above) --
    catches rare-path bugs (flagged elements, patching) the small sets miss."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = os.path.join(root, "profiles", "k1_bench.py")

    def digests(env):
        out = subprocess.run([sys.executable, script, "400000"], capture_output=True, text=True,
                             env={**os.environ, **env}, timeout=600, check=True).stdout
        return [line.split("sha=")[1].strip() for line in out.splitlines() if "sha=" in line]

    ref = digests({"QGNN_K1_GRP": "0"})
    assert len(ref) == 6
    assert digests({"QGNN_K1_GRP": "1"}) == ref
    assert digests({"QGNN_K1_GRP": "1", "QGNN_K1_EPL": "16"}) == ref
    assert digests({"QGNN_K1_GRP": "1", "QGNN_K1_YDOM": "0"}) == ref  # the x-domain form
