"""Python handle on the C++ GPU engine (trainer/engine.hpp's Engine, B200 edition).

    eng = Engine(graph, dims=[F, 256, 256, C], n_parts=8, bit_mode="adaptive")
    m = eng.run_epoch()          # dict: train_loss, val_acc, ..., ms_total

``graph`` is a dict with CSR ``adj_ptr`` (int64), ``adj`` (int32), ``features``
(float32/float64, n x F), ``labels`` (int32) and ``train``/``val``/``test``
masks (uint8), as produced by :func:`generate_planted` or the oracle's
reference generator.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import F32, F64, WIRE_GPU, WIRE_REF, check, lib

# input generation lives outside the product (shared by both bench arms)
from synth import generate_planted  # noqa: F401

BIT_MODES = {"fp": 0, "fixed": 1, "uniform": 2, "adaptive": 3}
KCLASSES = ["quant", "dequant", "spmm_fwd", "spmm_bwd", "partials", "gemm_fwd", "gemm_dgrad",
            "gemm_wgrad", "elemwise", "exchange"]


def partition_stats(g, owner, n_parts):
    out = np.zeros((n_parts, 5), np.int64)
    ptr, adj = g["adj_ptr"], g["adj"]
    own = np.ascontiguousarray(owner, np.uint32)
    check(lib.qgnn_partition_stats(ptr.ctypes.data, adj.ctypes.data, len(ptr) - 1,
                                   own.ctypes.data, n_parts, out.ctypes.data))
    return out  # per part: owned, central, marginal, halo, sum |remote_out|


def exchange_plan(g, owner, n_parts: int, world: int, rank: int, dim: int, bits: int = 8,
                  bwd: bool = False, layout: int = 0, dtype: str = "f32"):
    """Bytes this rank sends to / receives from every rank for one tensor key
    (qgnn_exchange_plan; the reference's pair_wire_bytes / negotiate_buffers,
    assigner/plan.hpp:90-154).  Returns (send[world], recv[world])."""
    ptr, adj = g["adj_ptr"], g["adj"]
    own = np.ascontiguousarray(owner, np.uint32)
    send = np.zeros(world, np.uint64)
    recv = np.zeros(world, np.uint64)
    check(lib.qgnn_exchange_plan(ptr.ctypes.data, adj.ctypes.data, len(ptr) - 1, own.ctypes.data,
                                 n_parts, world, rank, dim, bits, int(bwd), layout,
                                 1 if dtype == "f64" else 0, send.ctypes.data, recv.ctypes.data))
    return send, recv


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    check(lib.qgnn_nccl_unique_id(buf))
    return bytes(buf)


def load_dataset(path, device: Optional[int] = 0) -> dict:
    """The reference's dataset directory (load_dataset, cli/synth.hpp:184-205) through
    qgnn_dataset_load: CSR built on `device` (None: on the host), features as fp32
    (``features``) and as stored (``features_f64``); the dict feeds :class:`Engine`."""
    h = C.c_void_p()
    check(lib.qgnn_dataset_load(str(path).encode(), -1 if device is None else int(device),
                                C.byref(h)))
    try:
        a = _lib.DatasetArrays()
        check(lib.qgnn_dataset_arrays_get(h, C.byref(a)))
        n, e, f = a.nodes, a.nnz, a.feature_dim

        def arr(p, cnt, ct, dt):
            if cnt == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (cnt,)).astype(dt)

        return dict(adj_ptr=arr(a.adj_ptr, n + 1, C.c_int64, np.int64),
                    adj=arr(a.adj, e, C.c_int32, np.int32),
                    features=arr(a.features_f32, n * f, C.c_float, np.float32).reshape(n, f),
                    features_f64=arr(a.features, n * f, C.c_double, np.float64).reshape(n, f),
                    labels=arr(a.labels, n, C.c_int32, np.int32),
                    train=arr(a.train, n, C.c_uint8, np.uint8),
                    val=arr(a.val, n, C.c_uint8, np.uint8),
                    test=arr(a.test, n, C.c_uint8, np.uint8), classes=int(a.classes))
    finally:
        lib.qgnn_dataset_destroy(h)


def loopback_id(group: int) -> bytes:
    """Id for the in-process loopback transport (one thread per rank, one GPU)."""
    buf = (C.c_char * 128)()
    check(lib.qgnn_loopback_id(group, buf))
    return bytes(buf)


class Engine:
    def __init__(self, graph, dims: Sequence[int], n_parts: int, bit_mode: str = "fixed",
                 fixed_bits: int = 8, seed: int = 7, sage: bool = False, lam: float = 0.5,
                 group_size: int = 4, period: int = 50, lr: float = 0.01, theta: float = 3e-9,
                 gamma: float = 5e-5, dtype: str = "f32", layout: Optional[int] = None,
                 owner=None, rank: int = 0, world: int = 1, device: int = 0,
                 nccl_id: Optional[bytes] = None, kstats: bool = False, overlap: int = 1,
                 transport: str = "zero_copy", layer_norm: bool = False, dropout: float = 0.0):
        s = _lib.Settings()
        s.sage = int(sage)
        s.n_dims = len(dims)
        for i, d in enumerate(dims):
            s.dims[i] = int(d)
        s.bit_mode = BIT_MODES[bit_mode]
        s.fixed_bits = fixed_bits
        s.lambda_ = lam
        s.group_size = group_size
        s.period = period
        s.seed = seed
        s.n_parts = n_parts
        s.lr = lr
        s.theta = theta
        s.gamma = gamma
        s.dtype = F64 if dtype == "f64" else F32
        s.layout = (WIRE_REF if dtype == "f64" else WIRE_GPU) if layout is None else layout
        s.rank, s.world, s.device = rank, world, device
        s.overlap = int(overlap)
        s.transport = {"zero_copy": 0, "nccl": 1, "p2p": 2}[transport]
        s.kstats = int(kstats)
        s.layer_norm = int(layer_norm)
        s.dropout = float(dropout)
        self.settings = s
        self.dims = list(dims)
        self.np_dtype = np.float64 if dtype == "f64" else np.float32
        # a loaded dataset carries the stored f64 features next to the fp32 ones
        src = graph.get("features_f64", graph["features"]) if dtype == "f64" else graph["features"]
        feats = np.ascontiguousarray(src, self.np_dtype)
        self._keep = dict(
            ptr=np.ascontiguousarray(graph["adj_ptr"], np.int64),
            adj=np.ascontiguousarray(graph["adj"], np.int32), feats=feats,
            labels=np.ascontiguousarray(graph["labels"], np.int32),
            train=np.ascontiguousarray(graph["train"], np.uint8),
            val=np.ascontiguousarray(graph["val"], np.uint8),
            test=np.ascontiguousarray(graph["test"], np.uint8),
            owner=None if owner is None else np.ascontiguousarray(owner, np.uint32))
        k = self._keep
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_char * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        check(lib.qgnn_engine_create(
            C.byref(s), len(k["ptr"]) - 1, k["ptr"].ctypes.data, k["adj"].ctypes.data,
            feats.ctypes.data, k["labels"].ctypes.data, k["train"].ctypes.data,
            k["val"].ctypes.data, k["test"].ctypes.data,
            None if k["owner"] is None else k["owner"].ctypes.data,
            None if idbuf is None else C.cast(idbuf, C.c_void_p), C.byref(h)))
        self._h = h
        del self._keep["adj"]  # the engine keeps its own copies

    def close(self):
        if getattr(self, "_h", None):
            lib.qgnn_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def run_epoch(self) -> dict:
        m = _lib.EpochMetrics()
        check(lib.qgnn_engine_run_epoch(self._h, C.byref(m)))
        return m.as_dict()

    def set_kstats(self, on: bool) -> None:
        """Per-kernel event timing on/off (off: the epoch replays as a CUDA graph)."""
        check(lib.qgnn_engine_set_kstats(self._h, int(bool(on))))

    def launch_epoch(self) -> None:
        """Enqueue one epoch and return (pair with finish_epoch)."""
        check(lib.qgnn_engine_launch_epoch(self._h))

    def finish_epoch(self) -> dict:
        """Wait for the launched epoch; returns its metrics (loss read back)."""
        m = _lib.EpochMetrics()
        check(lib.qgnn_engine_finish_epoch(self._h, C.byref(m)))
        return m.as_dict()

    def set_features(self, feats):
        """Upload node features (n x F).  A pinned torch tensor (or a CUDA
        tensor) takes the fast path: asynchronous node-range copies that the
        next run_epoch consumes partition by partition as they land (keep the
        tensor alive until then); a numpy array is staged through pinned
        memory synchronously."""
        if hasattr(feats, "data_ptr"):
            assert feats.is_contiguous() and feats.element_size() == np.dtype(self.np_dtype).itemsize
            check(lib.qgnn_engine_set_features(self._h, C.c_void_p(feats.data_ptr())))
            return
        f = np.ascontiguousarray(feats, self.np_dtype)
        check(lib.qgnn_engine_set_features(self._h, f.ctypes.data))

    def weights(self):
        out = []
        for l in range(len(self.dims) - 1):
            w = np.zeros((self.dims[l], self.dims[l + 1]), self.np_dtype)
            check(lib.qgnn_engine_get_weights(self._h, l, w.ctypes.data))
            out.append(w)
        return out

    def set_weights(self, ws):
        for l, w in enumerate(ws):
            w = np.ascontiguousarray(w, self.np_dtype)
            check(lib.qgnn_engine_set_weights(self._h, l, w.ctypes.data))

    def info(self) -> dict:
        out = np.zeros(6, np.int64)
        check(lib.qgnn_engine_info(self._h, out.ctypes.data))
        return dict(messages_per_tensor=int(out[0]), n_parts=int(out[1]),
                    parts_on_rank=int(out[2]), max_owned=int(out[3]), max_halo=int(out[4]),
                    launches_last_epoch=int(out[5]))

    def kernel_stats(self) -> dict:
        out = np.zeros(4 * len(KCLASSES))
        n = lib.qgnn_engine_kernel_stats(self._h, out.ctypes.data, len(out))
        if n < 0:
            check(-n)
        return {KCLASSES[i]: dict(ms=out[4 * i], launches=int(out[4 * i + 1]),
                                  bytes=out[4 * i + 2], gathered=out[4 * i + 3])
                for i in range(n)}
