"""The reference's on-disk dataset (SURVEY.md §8f rank 3 loader): qgnn_dataset_load
against the reference's own save_dataset / load_dataset (cli/synth.hpp:153-205,
graph.hpp:59-200) through oracle/_ref.  CPU tests use the host CSR build; the
GPU tests the radix-sort build on the device and an engine trained from a loaded
directory."""
import os

import numpy as np
import pytest

from oracle import ref
from paper_2306_01381_b200 import _lib
from paper_2306_01381_b200.engine import Engine, load_dataset


def _same(got, exp):
    assert np.array_equal(got["adj_ptr"], exp["adj_ptr"])
    assert np.array_equal(got["adj"], exp["adj"])
    assert np.array_equal(got["features_f64"], exp["features"])
    assert np.array_equal(got["features"], exp["features"].astype(np.float32))
    for k in ("labels", "train", "val", "test"):
        assert np.array_equal(got[k], exp[k]), k


@pytest.fixture(scope="module")
def saved(tmp_path_factory):
    d = tmp_path_factory.mktemp("cite")
    g = ref.generate_and_save(d, kind="cite", nodes=3000, classes=5, feature_dim=12,
                              attach_edges=6, seed=3)
    return d, g


def test_load_matches_reference_host(saved):
    d, g = saved
    exp = ref.load_dataset(d)
    got = load_dataset(d, device=None)
    _same(got, exp)
    assert got["classes"] == 5
    # and the graph the reference generated in memory
    assert np.array_equal(got["adj"], g["adj"]) and np.array_equal(got["adj_ptr"], g["adj_ptr"])


def _edge_variants(d, text):
    (d / "edges.txt").write_text(text)


def test_edge_list_semantics_host(saved, tmp_path):
    """Comments, blank lines, duplicates, both directions and self loops: the same
    symmetric, deduplicated, sorted CSR as build_graph (graph.hpp:59-78)."""
    d, _ = saved
    for f in os.listdir(d):
        (tmp_path / f).write_bytes((d / f).read_bytes())
    _edge_variants(tmp_path, "# header\n0 1\n1 0\n\n2 2\n5 3   # trailing comment\n 7\t9\n0 1\n"
                             "2999 0\n")
    exp = ref.load_dataset(tmp_path)
    got = load_dataset(tmp_path, device=None)
    _same(got, exp)


@pytest.mark.parametrize("case,err,msg", [
    ("edges", _lib.IoError, "expected two node ids"),
    ("range", _lib.InvalidArgument, "edge endpoint out of range"),
    ("features", _lib.IoError, "truncated payload"),
    ("labels", _lib.IoError, "label count mismatch"),
    ("masks", _lib.InvalidArgument, "overlapping masks"),
    ("meta", _lib.IoError, "cannot open dataset meta"),
])
def test_load_errors_host(saved, tmp_path, case, err, msg):
    d, _ = saved
    for f in os.listdir(d):
        (tmp_path / f).write_bytes((d / f).read_bytes())
    if case == "edges":
        (tmp_path / "edges.txt").write_text("0 1\n2\n")
    elif case == "range":
        (tmp_path / "edges.txt").write_text("0 1\n0 3000\n")
    elif case == "features":
        b = (tmp_path / "features.bin").read_bytes()
        (tmp_path / "features.bin").write_bytes(b[:-8])
    elif case == "labels":
        (tmp_path / "labels.txt").write_text("0\n1\n")
    elif case == "masks":
        (tmp_path / "val_mask.txt").write_text((tmp_path / "train_mask.txt").read_text())
    elif case == "meta":
        os.remove(tmp_path / "meta.json")
    with pytest.raises(err, match=msg):
        load_dataset(tmp_path, device=None)
    if case != "meta":  # the reference rejects the same directory
        with pytest.raises(Exception):
            ref.load_dataset(tmp_path)


@pytest.mark.gpu
def test_load_matches_reference_gpu(cuda, saved):
    d, _ = saved
    _same(load_dataset(d, device=0), ref.load_dataset(d))


@pytest.mark.gpu
def test_gpu_csr_build_random_edges(cuda, tmp_path, saved):
    """1M random edges with duplicates, reversed pairs and self loops: device and
    host builds identical."""
    d, _ = saved
    for f in os.listdir(d):
        (tmp_path / f).write_bytes((d / f).read_bytes())
    rs = np.random.default_rng(5)
    e = rs.integers(0, 3000, (1_000_000, 2))
    e[::50, 1] = e[::50, 0]
    (tmp_path / "edges.txt").write_text("\n".join(f"{u} {v}" for u, v in e) + "\n")
    a = load_dataset(tmp_path, device=0)
    b = load_dataset(tmp_path, device=None)
    assert np.array_equal(a["adj_ptr"], b["adj_ptr"]) and np.array_equal(a["adj"], b["adj"])


@pytest.mark.gpu
def test_engine_from_loaded_dataset(cuda, saved):
    """Training from a loaded directory is the same run as from the reference's
    in-memory arrays (f64: bit-identical losses)."""
    d, g = saved
    loaded = load_dataset(d, device=0)
    kw = dict(dims=[12, 16, 5], n_parts=2, bit_mode="fixed", fixed_bits=8, seed=7, dtype="f64")
    a = Engine(loaded, **kw)
    b = Engine(g, **kw)
    la = [a.run_epoch()["train_loss"] for _ in range(3)]
    lb = [b.run_epoch()["train_loss"] for _ in range(3)]
    a.close()
    b.close()
    assert la == lb
