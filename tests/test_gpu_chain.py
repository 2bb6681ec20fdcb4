"""LayerNorm and dropout (TrainSettings::layer_norm / dropout, engine.hpp:42-43;
model.hpp:62-153) against the compiled reference Engine on the same inputs.

The dropout masks are drawn on the GPU from the reference's own coordinates
(RngStream(seed).fork({0x4, epoch, layer, device}).fork(row), engine.hpp:600,
model.hpp:114-119), so the fp64 engine must reproduce the reference's losses to
1e-12 and its accuracies exactly; the production fp32 engine (3xTF32 GEMMs,
transform-first last layer, fused packed halo) within the north-star
tolerances (loss 1e-4 relative, accuracy 0.3 %)."""
import numpy as np
import pytest

from oracle import ref
from paper_2306_01381_b200.engine import Engine
from synth import generate_planted

pytestmark = pytest.mark.gpu

CASES = [(True, 0.0), (False, 0.3), (True, 0.5)]


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


@pytest.fixture(scope="module")
def cite():
    return ref.generate_dataset(kind="cite", nodes=1500, classes=6, feature_dim=32,
                                attach_edges=5, seed=4)


def _engine(g, dims, parts, epochs, **kw):
    eng = Engine(g, dims, n_parts=parts, **kw)
    out = [eng.run_epoch() for _ in range(epochs)]
    w = np.concatenate([x.reshape(-1) for x in eng.weights()])
    eng.close()
    return out, w


@pytest.mark.parametrize("ln,dropout", CASES)
def test_chain_f64_engine_matches_reference(cuda, cite, ln, dropout):
    dims = [32, 48, 48, 6]
    ep, w_ref = ref.engine_run(cite, dims, 3, bit_mode=1, fixed_bits=8, epochs=4, seed=9,
                               threads=True, layer_norm=ln, dropout=dropout)
    got, w = _engine(cite, dims, 3, 4, bit_mode="fixed", fixed_bits=8, seed=9, dtype="f64",
                     owner=None, layer_norm=ln, dropout=dropout)
    for e, m in enumerate(got):
        assert _rel(m["train_loss"], ep[e, 0]) < 1e-12, (e, m["train_loss"], ep[e, 0])
        assert m["val_acc"] == ep[e, 1] and m["test_acc"] == ep[e, 2], e
        assert m["ref_bytes_total"] == ep[e, 3], e
    assert np.allclose(w, w_ref, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("ln,dropout", CASES)
def test_chain_f32_engine_within_tolerance(cuda, cite, ln, dropout):
    dims = [32, 48, 48, 6]
    ep, _ = ref.engine_run(cite, dims, 3, bit_mode=1, fixed_bits=8, epochs=4, seed=9,
                           threads=True, layer_norm=ln, dropout=dropout)
    got, _ = _engine(cite, dims, 3, 4, bit_mode="fixed", fixed_bits=8, seed=9, dtype="f32",
                     owner=None, layer_norm=ln, dropout=dropout)
    for e, m in enumerate(got):
        assert _rel(m["train_loss"], ep[e, 0]) < 1e-4, (e, m["train_loss"], ep[e, 0])
        assert abs(m["val_acc"] - ep[e, 1]) <= 0.003, (e, m["val_acc"], ep[e, 1])
        assert abs(m["test_acc"] - ep[e, 2]) <= 0.003, (e, m["test_acc"], ep[e, 2])


def test_chain_production_shape_f32(cuda):
    """1/64 config-4 sample (256/100/47 widths, P=8, adaptive): LayerNorm + dropout 0.1
    through the production kernels, the transform-first last layer included."""
    g = generate_planted(2449029 // 64, 61859140 // 64, 100, 47, 8, 0.0085, gamma=2.8, seed=1)
    kw = dict(seed=7, group_size=2000, period=2, theta=1.0 / (900e9 * 8), gamma=2e-5)
    gg = dict(g)
    gg["features"] = g["features"].astype(np.float64)
    dims = [100, 256, 256, 47]
    ep, _ = ref.engine_run(gg, dims, 8, bit_mode=3, epochs=3, threads=True, owner=g["owner"],
                           layer_norm=True, dropout=0.1, **kw)
    got, _ = _engine(g, dims, 8, 3, bit_mode="adaptive", dtype="f32", owner=g["owner"],
                     layer_norm=True, dropout=0.1, **kw)
    plain, _ = _engine(g, dims, 8, 1, bit_mode="adaptive", dtype="f32", owner=g["owner"], **kw)
    assert plain[0]["train_loss"] != got[0]["train_loss"]  # the chain is really on
    for e, m in enumerate(got):
        assert _rel(m["train_loss"], ep[e, 0]) < 1e-4, (e, m["train_loss"], ep[e, 0])
        assert abs(m["val_acc"] - ep[e, 1]) <= 0.003, (e, m["val_acc"], ep[e, 1])
        assert (m["msgs_b2"], m["msgs_b4"], m["msgs_b8"]) == tuple(ep[e, 4:7]), e


def test_dropout_out_of_range_is_rejected():
    from paper_2306_01381_b200 import InvalidArgument
    g = generate_planted(200, 800, 8, 2, 2, 0.05, seed=3)
    with pytest.raises((InvalidArgument, Exception)):
        Engine(g, [8, 8, 2], n_parts=2, dropout=1.0)
