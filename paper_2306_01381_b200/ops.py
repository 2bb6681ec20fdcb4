"""Host mirror of the reference operator API over the C-ABI (torch tensors for device memory).

Each function names the reference function it stands in for.  Arguments are
CUDA tensors; the kernels run on the current torch stream and the context's
device error word is checked before returning, so failures surface as the
reference's exception types (``DecodeError``, ``InvalidArgument`` ...).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import F32, F64, WIRE_GPU, WIRE_REF, check, lib

_CTX = {}


def ctx(device: Optional[int] = None):
    """Per-device qgnn_ctx (error word + scratch)."""
    if device is None:
        device = torch.cuda.current_device()
    if device not in _CTX:
        h = C.c_void_p()
        check(lib.qgnn_ctx_create(device, C.byref(h)))
        _CTX[device] = h
    return _CTX[device]


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise _lib.InvalidArgument(f"unsupported dtype {t.dtype}")


def sync_check(device: Optional[int] = None) -> None:
    check(lib.qgnn_ctx_check(ctx(device), _stream()))


# ---- rng.hpp ------------------------------------------------------------------
def rng_key(seed: int, *coords: int) -> int:
    """Key of RngStream(seed).fork(c0).fork(c1)... (rng.hpp:15-28)."""
    k = lib.qgnn_rng_seed_key(seed & (2**64 - 1))
    for c in coords:
        k = lib.qgnn_rng_fork(k, c & (2**64 - 1))
    return k


def chunk_wire_bytes(count: int, bits: int, layout: int = WIRE_GPU, dtype: int = F32) -> int:
    return int(lib.qgnn_chunk_wire_bytes(count, bits, layout, dtype))


def wire_layout(bits: np.ndarray, dim: int, layout: int = WIRE_GPU, dtype: int = F32):
    """encode_message_set wire order (codec.hpp:56-69): (wire_pos, offsets, total)."""
    bits = np.ascontiguousarray(bits, np.int32)
    n = len(bits)
    pos = np.zeros(max(1, n), np.int64)
    off = np.zeros(max(1, n), np.uint64)
    tot = C.c_uint64()
    check(lib.qgnn_wire_layout(bits.ctypes.data, n, dim, layout, dtype, pos.ctypes.data,
                               off.ctypes.data, C.byref(tot)))
    return pos[:n], off[:n], tot.value


# ---- codec.hpp / quant.hpp ----------------------------------------------------------
def quantize_pack(values, rows, ids, bits, offsets, set_keys, out, layout=WIRE_GPU, set_of=None,
                  win_lo=None, win_hi=None, check_errors=True, envelope=0):
    """K1 over arbitrary (row, id, width, offset) message lists."""
    dim = values.shape[1]
    check(lib.qgnn_quantize_pack(ctx(), _ptr(values), _dtype(values), values.stride(0), dim,
                                 rows.numel(), _ptr(rows), _ptr(ids), _ptr(bits), _ptr(offsets),
                                 _ptr(set_of), _ptr(set_keys), layout, _ptr(out), _ptr(win_lo),
                                 _ptr(win_hi), envelope, _stream()))
    if check_errors:
        sync_check()
    return out


def encode_message_set(values: torch.Tensor, rows, ids, bits, set_key: int,
                       layout: int = WIRE_GPU):
    """encode_message_set (codec.hpp:41-72) on the GPU.

    ``rows``/``ids``/``bits`` are host arrays in caller order.  Returns the wire
    bytes (CUDA uint8 tensor) and the retrieval index (wire order) as numpy
    arrays: (pos -> caller index, bits, offset).
    """
    dev = values.device
    ids_np = np.ascontiguousarray(ids, np.uint32)
    if len(np.unique(ids_np)) != len(ids_np):
        raise _lib.InvalidArgument("encode_message_set: duplicate message ids")
    bits_np = np.ascontiguousarray(bits, np.int32)
    pos, off, total = wire_layout(bits_np, values.shape[1], layout, _dtype(values))
    out = torch.zeros(max(total, 16), dtype=torch.uint8, device=dev)
    rows_t = torch.as_tensor(np.ascontiguousarray(rows, np.int32), device=dev)
    ids_t = torch.as_tensor(ids_np.view(np.int32), device=dev)
    bits_t = torch.as_tensor(bits_np.astype(np.uint8), device=dev)
    off_t = torch.as_tensor(off.view(np.int64), device=dev)
    keys = torch.as_tensor(np.array([set_key], np.uint64).view(np.int64), device=dev)
    quantize_pack(values, rows_t, ids_t, bits_t, off_t, keys, out, layout=layout)
    return out[:total], dict(pos=pos, bits=bits_np[pos], off=off[pos], total=total)


def dequant_scatter(wire, bits, offsets, dim, out, dst_rows=None, accumulate=False,
                    layout=WIRE_GPU, check_errors=True, expect_envelope=None):
    """K3: decode_message_set (codec.hpp:80-96) fused with the halo scatter."""
    n = bits.numel()
    check(lib.qgnn_dequant_scatter(ctx(), _ptr(wire), n, dim, _ptr(bits), _ptr(offsets), layout,
                                   _ptr(dst_rows), int(accumulate), _ptr(out), _dtype(out),
                                   out.stride(0), _ptr(expect_envelope), _stream()))
    if check_errors:
        sync_check()
    return out


def validate_index(bits, offsets, dim, n_bytes: int, total: Optional[int] = None,
                   layout: int = WIRE_GPU, dtype: int = F32) -> None:
    """decode_message_set's index checks (qgnn_decode_validate, codec.hpp:82-95):
    raises DecodeError like the reference."""
    b = np.ascontiguousarray(bits, np.uint8)
    o = np.ascontiguousarray(offsets, np.uint64)
    d = np.full(len(b), dim, np.uint64)
    check(lib.qgnn_decode_validate(b.ctypes.data, o.ctypes.data, d.ctypes.data, len(b), layout,
                                   dtype, n_bytes if total is None else total, n_bytes))


def decode_message_set(wire: torch.Tensor, bits, offsets, dim: int, dtype=torch.float32,
                       layout: int = WIRE_GPU, total: Optional[int] = None):
    """decode_message_set: rows in index (wire) order.  ``total`` is the
    index's total_bytes (default: the wire length); the index is validated on
    the host first, each chunk against its entry on the device."""
    dev = wire.device
    n = len(bits)
    validate_index(bits, offsets, dim, wire.numel(), total, layout,
                   F64 if dtype == torch.float64 else F32)
    out = torch.zeros((max(1, n), dim), dtype=dtype, device=dev)
    bits_t = torch.as_tensor(np.ascontiguousarray(bits, np.uint8), device=dev)
    off_t = torch.as_tensor(np.ascontiguousarray(offsets, np.uint64).view(np.int64), device=dev)
    dequant_scatter(wire, bits_t, off_t, dim, out, layout=layout)
    return out[:n]


# ---- aggregate.hpp ---------------------------------------------------------------
def csr_aggregate(x, ptr_a, col_a, alpha_a, out, self_alpha=None, y=None, ptr_b=None, col_b=None,
                  alpha_b=None, rows=None, row_begin=0, n_rows=None):
    """K4 (see qgnn_csr_aggregate)."""
    dim = x.shape[1]
    if n_rows is None:
        n_rows = rows.numel() if rows is not None else out.shape[0] - row_begin
    check(lib.qgnn_csr_aggregate(ctx(), _dtype(x), dim, _ptr(x), x.stride(0), _ptr(y),
                                 y.stride(0) if y is not None else 0, _ptr(self_alpha),
                                 _ptr(ptr_a), _ptr(col_a), _ptr(alpha_a), _ptr(ptr_b),
                                 _ptr(col_b), _ptr(alpha_b), _ptr(rows), row_begin, n_rows,
                                 _ptr(out), out.stride(0), _stream()))
    return out


class SpmmPlan:
    """Production fp32 K4 over one CSR row range (qgnn_spmm_plan_*): the
    engine's kernels, hub segmentation and degree-sorted narrow rows.
    ``ptr_a``/``ptr_b`` are host (numpy int64) row pointers; runs take device
    tensors."""

    def __init__(self, ptr_a, row_begin, n_rows, max_dim, ptr_b=None, hub_deg=128):
        self._pa = np.ascontiguousarray(ptr_a, np.int64)
        self._pb = None if ptr_b is None else np.ascontiguousarray(ptr_b, np.int64)
        h = C.c_void_p()
        check(lib.qgnn_spmm_plan_create(ctx(), self._pa.ctypes.data,
                                        None if self._pb is None else self._pb.ctypes.data,
                                        row_begin, n_rows, max_dim, hub_deg, C.byref(h)))
        self._h = h

    def run(self, dim, x, ptr_a, col_a, alpha_a, out, self_alpha=None, y=None, ptr_b=None,
            col_b=None, alpha_b=None, mask=None):
        check(lib.qgnn_spmm_plan_run(self._h, dim, _ptr(x), x.stride(0), _ptr(y),
                                     y.stride(0) if y is not None else 0, _ptr(self_alpha),
                                     _ptr(ptr_a), _ptr(col_a), _ptr(alpha_a), _ptr(ptr_b),
                                     _ptr(col_b), _ptr(alpha_b), _ptr(mask),
                                     mask.stride(0) if mask is not None else 0, _ptr(out),
                                     out.stride(0), _stream()))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib.qgnn_spmm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


# ---- exchange.hpp / engine.hpp mailbox ------------------------------------------------
class Comm:
    """One rank of an exchange group (qgnn_comm_*): NCCL (id from
    engine.nccl_unique_id(), or None for world 1) or the in-process loopback
    transport (engine.loopback_id(group), ranks as threads)."""

    def __init__(self, world: int = 1, rank: int = 0, id128: Optional[bytes] = None,
                 device: Optional[int] = None):
        if device is None:
            device = torch.cuda.current_device()
        idbuf = None if id128 is None else (C.c_char * 128).from_buffer_copy(id128)
        h = C.c_void_p()
        check(lib.qgnn_comm_create(None if idbuf is None else C.cast(idbuf, C.c_void_p), world,
                                   rank, device, C.byref(h)))
        self._h, self.world, self.rank = h, world, rank

    def exchange(self, send: torch.Tensor, send_off, send_bytes, recv: torch.Tensor, recv_off,
                 recv_bytes):
        """Grouped point-to-point all-to-all-v (qgnn_exchange) on the current stream."""
        arr = [np.ascontiguousarray(a, np.uint64) for a in (send_off, send_bytes, recv_off,
                                                           recv_bytes)]
        assert all(len(a) == self.world for a in arr)
        check(lib.qgnn_exchange(self._h, _ptr(send), arr[0].ctypes.data, arr[1].ctypes.data,
                                _ptr(recv), arr[2].ctypes.data, arr[3].ctypes.data, _stream()))
        return recv

    def close(self):
        if getattr(self, "_h", None):
            lib.qgnn_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


# ---- model.hpp / matrix.hpp ---------------------------------------------------------
def dense_forward(a, w, out, relu=True, rows=None, row_begin=0, n_rows=None):
    if n_rows is None:
        n_rows = rows.numel() if rows is not None else a.shape[0] - row_begin
    check(lib.qgnn_dense_forward(ctx(), _dtype(a), _ptr(a), a.stride(0), _ptr(w), w.shape[0],
                                 w.shape[1], _ptr(rows), row_begin, n_rows, int(relu), _ptr(out),
                                 out.stride(0), _stream()))
    return out


def dense_input_grad(dz, w, out, rows=None, row_begin=0, n_rows=None):
    if n_rows is None:
        n_rows = rows.numel() if rows is not None else dz.shape[0] - row_begin
    check(lib.qgnn_dense_input_grad(ctx(), _dtype(dz), _ptr(dz), dz.stride(0), _ptr(w),
                                    w.shape[0], w.shape[1], _ptr(rows), row_begin, n_rows,
                                    _ptr(out), out.stride(0), _stream()))
    return out


def dense_weight_grad(a, b, out, rows=None, row_begin=0, n_rows=None, accumulate=False):
    if n_rows is None:
        n_rows = rows.numel() if rows is not None else a.shape[0] - row_begin
    check(lib.qgnn_dense_weight_grad(ctx(), _dtype(a), _ptr(a), a.stride(0), _ptr(b),
                                     b.stride(0), a.shape[1], b.shape[1], _ptr(rows), row_begin,
                                     n_rows, int(accumulate), _ptr(out), _stream()))
    return out


def relu_backward(act, dh, dz, row_begin=0, n_rows=None):
    if n_rows is None:
        n_rows = act.shape[0] - row_begin
    check(lib.qgnn_relu_backward(ctx(), _dtype(act), _ptr(act), act.stride(0), _ptr(dh),
                                 dh.stride(0), act.shape[1], row_begin, n_rows, _ptr(dz),
                                 dz.stride(0), _stream()))
    return dz


def masked_ce(logits, labels, rows, inv_denom, grad):
    acc = torch.zeros(1, dtype=torch.float64, device=logits.device)
    check(lib.qgnn_masked_ce(ctx(), _dtype(logits), _ptr(logits), logits.stride(0),
                             logits.shape[1], _ptr(labels), _ptr(rows), rows.numel(), inv_denom,
                             _ptr(grad), grad.stride(0), _ptr(acc), _stream()))
    sync_check()
    return float(acc.item())


def count_correct(logits, labels, rows):
    acc = torch.zeros(1, dtype=torch.int64, device=logits.device)
    check(lib.qgnn_count_correct(ctx(), _dtype(logits), _ptr(logits), logits.stride(0),
                                 logits.shape[1], _ptr(labels), _ptr(rows), rows.numel(),
                                 _ptr(acc), _stream()))
    return int(acc.item())


def adam_step(p, m, v, g, t, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8):
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    check(lib.qgnn_adam_step(ctx(), _dtype(p), _ptr(p), _ptr(m), _ptr(v), _ptr(g), p.numel(), lr,
                             beta1, beta2, eps, bc1, bc2, _stream()))
    return p


# ---- graphcore/partition.hpp, tensorops/aggregate.hpp, assigner/plan.hpp (host) -------------
def _partition_handles(adj_ptr, adj, owner, n_parts, gpu_device):
    hs = (C.c_void_p * n_parts)()
    if gpu_device is None:
        check(lib.qgnn_partitions_from_owner(adj_ptr.ctypes.data, adj.ctypes.data, len(owner),
                                             owner.ctypes.data, n_parts, hs))
    else:  # consumer sets on the device
        check(lib.qgnn_partitions_from_owner_gpu(adj_ptr.ctypes.data, adj.ctypes.data,
                                                 len(owner), owner.ctypes.data, n_parts,
                                                 gpu_device, hs))
    return hs


def partitions_from_owner(adj_ptr, adj, owner, n_parts: int, gpu_device: Optional[int] = None):
    """partitions_from_owner (partition.hpp:39-84) through the C-ABI: one dict
    per device with owned / central / marginal and remote_in[q] / remote_out[q]
    (ascending node ids, like Partition).  gpu_device: build on that GPU
    (qgnn_partitions_from_owner_gpu) instead of the host."""
    adj_ptr = np.ascontiguousarray(adj_ptr, np.int64)
    adj = np.ascontiguousarray(adj, np.int32)
    owner = np.ascontiguousarray(owner, np.uint32)
    hs = _partition_handles(adj_ptr, adj, owner, n_parts, gpu_device)

    def lst(h, which, q=0):
        p, n = C.c_void_p(), C.c_int64()
        check(lib.qgnn_partition_list(h, which, q, C.byref(p), C.byref(n)))
        if n.value == 0:
            return np.zeros(0, np.uint32)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint32)), (n.value,)).copy()

    out = []
    try:
        for h in hs:
            out.append(dict(owned=lst(h, 0), central=lst(h, 1), marginal=lst(h, 2),
                            remote_in=[lst(h, 3, q) for q in range(n_parts)],
                            remote_out=[lst(h, 4, q) for q in range(n_parts)]))
    finally:
        for h in hs:
            lib.qgnn_partition_destroy(h)
    return out


def agg_view(adj_ptr, adj, owner, n_parts: int, device: int, sage: bool = False,
             gpu_device: Optional[int] = None):
    """DeviceAggView::build (aggregate.hpp:41-89) for `device` of the owner map,
    reference row / slot order, as numpy arrays.  gpu_device: partitions and
    view built on that GPU (qgnn_*_gpu) instead of the host."""
    adj_ptr = np.ascontiguousarray(adj_ptr, np.int64)
    adj = np.ascontiguousarray(adj, np.int32)
    owner = np.ascontiguousarray(owner, np.uint32)
    hs = _partition_handles(adj_ptr, adj, owner, n_parts, gpu_device)
    view = C.c_void_p()
    try:
        if gpu_device is None:
            check(lib.qgnn_agg_view_build(adj_ptr.ctypes.data, adj.ctypes.data, len(owner),
                                          owner.ctypes.data, hs[device], int(sage),
                                          C.byref(view)))
        else:
            check(lib.qgnn_agg_view_build_gpu(adj_ptr.ctypes.data, adj.ctypes.data, len(owner),
                                              owner.ctypes.data, hs[device], int(sage),
                                              gpu_device, C.byref(view)))
    finally:
        for h in hs:
            lib.qgnn_partition_destroy(h)
    try:
        a = _lib.AggViewArrays()
        check(lib.qgnn_agg_view_arrays_get(view, C.byref(a)))

        def arr(ptr, n, ct, dt):
            if n == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), (n,)).astype(dt)

        no, nr, ln, rn = a.num_owned, a.num_remote, a.local_nnz, a.remote_nnz
        return dict(num_owned=no, num_remote=nr,
                    self_alpha=arr(a.self_alpha, no, C.c_double, np.float64),
                    local_ptr=arr(a.local_ptr, no + 1, C.c_int64, np.int64),
                    local_row=arr(a.local_row, ln, C.c_uint32, np.int64),
                    local_alpha_fwd=arr(a.local_alpha_fwd, ln, C.c_double, np.float64),
                    local_alpha_bwd=arr(a.local_alpha_bwd, ln, C.c_double, np.float64),
                    remote_ptr=arr(a.remote_ptr, no + 1, C.c_int64, np.int64),
                    remote_slot=arr(a.remote_slot, rn, C.c_uint32, np.int64),
                    remote_alpha=arr(a.remote_alpha, rn, C.c_double, np.float64),
                    slot_node=arr(a.slot_node, nr, C.c_uint32, np.uint32),
                    slot_owner=arr(a.slot_owner, nr, C.c_uint32, np.uint32),
                    device_slot_offset=arr(a.device_slot_offset, a.n_parts + 1, C.c_int64,
                                           np.int64),
                    central=arr(a.central_rows, a.n_central, C.c_uint32, np.int64),
                    marginal=arr(a.marginal_rows, a.n_marginal, C.c_uint32, np.int64))
    finally:
        lib.qgnn_agg_view_destroy(view)


def plan_bits_for(ids, bits, query):
    """BitWidthPlan::Lookup::bits_for (plan.hpp:60-72) over one pair's sorted entries."""
    ids = np.ascontiguousarray(ids, np.uint32)
    bits = np.ascontiguousarray(bits, np.int32)
    query = np.ascontiguousarray(query, np.uint32)
    out = np.zeros(max(1, len(query)), np.int32)
    check(lib.qgnn_plan_bits_for(ids.ctypes.data, bits.ctypes.data, len(ids), query.ctypes.data,
                                 len(query), out.ctypes.data))
    return out[:len(query)]
