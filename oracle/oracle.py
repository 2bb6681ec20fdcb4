"""ctypes/numpy front end for the two oracle libraries (test infrastructure only)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(_HERE, "_build", "libqgnn_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libqgnn_ref.so")

PHI = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def build() -> None:
    """Compile the C restatement and (when /root/reference exists) the reference shim."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _u64(x):
    return C.c_uint64(int(x) & M64)


class _Port:
    """The C restatement (oracle/qgnn_oracle.c)."""

    def __init__(self):
        if not os.path.exists(PORT_SO):
            build()
        L = C.CDLL(PORT_SO)
        self.L = L
        for n in ("qo_mix", "qo_seed_key"):
            getattr(L, n).restype = C.c_uint64
            getattr(L, n).argtypes = [C.c_uint64]
        for n in ("qo_fork", "qo_draw_u64"):
            getattr(L, n).restype = C.c_uint64
            getattr(L, n).argtypes = [C.c_uint64, C.c_uint64]
        L.qo_draw_double.restype = C.c_double
        L.qo_draw_double.argtypes = [C.c_uint64, C.c_uint64]
        L.qo_next_below.restype = C.c_uint64
        L.qo_next_below.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_uint64]
        L.qo_next_gaussian.restype = C.c_double
        L.qo_next_gaussian.argtypes = [C.c_uint64, C.POINTER(C.c_uint64)]
        L.qo_packed_bytes.restype = C.c_uint64
        L.qo_packed_bytes.argtypes = [C.c_uint64, C.c_int]
        L.qo_chunk_wire_bytes.restype = C.c_uint64
        L.qo_chunk_wire_bytes.argtypes = [C.c_uint64, C.c_int]
        L.qo_quantize.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]
        L.qo_pack.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        L.qo_unpack.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_void_p]
        L.qo_dequantize.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_double,
                                    C.c_void_p]
        L.qo_encode_message_set.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        L.qo_encoded_size.restype = C.c_uint64
        L.qo_encoded_size.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.qo_decode_message_set.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                            C.c_uint64]
        L.qo_aggregate_rows.argtypes = [C.c_void_p] * 9 + [C.c_uint64, C.c_void_p, C.c_uint64,
                                                           C.c_void_p]
        L.qo_backward_remote_partials.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.c_void_p,
                                                                     C.c_uint64, C.c_void_p]
        L.qo_layer_forward_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                            C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                            C.c_void_p]
        L.qo_layer_backward_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                             C.c_uint64, C.c_int, C.c_void_p]
        L.qo_input_grad_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                         C.c_void_p, C.c_uint64, C.c_void_p]
        L.qo_matmul_transa.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                       C.c_uint64, C.c_void_p]
        L.qo_masked_ce_partial.restype = C.c_double
        L.qo_masked_ce_partial.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                           C.c_uint64, C.c_double, C.c_void_p]
        L.qo_adam_step.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.c_uint64, C.c_double,
                                                      C.c_double, C.c_double, C.c_double]
        L.qo_compute_coeffs.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                        C.c_void_p]

    # rng ---------------------------------------------------------------
    def seed_key(self, seed):
        return self.L.qo_seed_key(_u64(seed))

    def fork(self, key, *coords):
        for c in coords:
            key = self.L.qo_fork(_u64(key), _u64(c))
        return key

    def stream(self, seed, *coords):
        return self.fork(self.seed_key(seed), *coords)

    def draw_u64(self, key, ctr):
        return self.L.qo_draw_u64(_u64(key), _u64(ctr))

    def draw_double(self, key, ctr):
        return self.L.qo_draw_double(_u64(key), _u64(ctr))

    def gaussians(self, key, n):
        ctr = C.c_uint64(0)
        return np.array([self.L.qo_next_gaussian(_u64(key), C.byref(ctr)) for _ in range(n)])

    # quant -------------------------------------------------------------
    def packed_bytes(self, n, b):
        return int(self.L.qo_packed_bytes(n, b))

    def quantize(self, h, b, key):
        h = np.ascontiguousarray(h, dtype=np.float64)
        out = np.zeros(max(1, self.packed_bytes(len(h), b)), np.uint8)
        s, z = C.c_double(), C.c_double()
        st = self.L.qo_quantize(_p(h), len(h), b, _u64(key), C.byref(s), C.byref(z), _p(out))
        if st:
            raise ValueError(f"quantize: status {st}")
        return s.value, z.value, out[: self.packed_bytes(len(h), b)]

    def pack(self, codes, b):
        codes = np.ascontiguousarray(codes, dtype=np.uint32)
        out = np.zeros(max(1, self.packed_bytes(len(codes), b)), np.uint8)
        if self.L.qo_pack(_p(codes), len(codes), b, _p(out)):
            raise ValueError("pack")
        return out[: self.packed_bytes(len(codes), b)]

    def unpack(self, payload, b, n):
        payload = np.ascontiguousarray(payload, dtype=np.uint8)
        out = np.zeros(n, np.uint32)
        if self.L.qo_unpack(_p(payload), b, n, _p(out)):
            raise ValueError("unpack")
        return out

    def dequantize(self, payload, b, n, scale, zero):
        payload = np.ascontiguousarray(payload, dtype=np.uint8)
        out = np.zeros(n, np.float64)
        self.L.qo_dequantize(_p(payload), b, n, scale, zero, _p(out))
        return out

    def chunk_wire_bytes(self, n, b):
        return int(self.L.qo_chunk_wire_bytes(n, b))

    def encode_message_set(self, values, rows, ids, bits, set_key):
        values = np.ascontiguousarray(values, dtype=np.float64)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        bits = np.ascontiguousarray(bits, dtype=np.int32)
        n, dim = len(ids), values.shape[1]
        size = int(self.L.qo_encoded_size(_p(bits), n, dim))
        out = np.zeros(max(1, size), np.uint8)
        pos = np.zeros(max(1, n), np.int64)
        off = np.zeros(max(1, n), np.uint64)
        st = self.L.qo_encode_message_set(_p(values), values.shape[1], _p(rows), _p(ids),
                                          _p(bits), n, dim, _u64(set_key), _p(out), _p(pos),
                                          _p(off))
        if st:
            raise ValueError(f"encode_message_set: status {st}")
        return out[:size], pos[:n], off[:n]

    def decode_message_set(self, wire, e_bits, e_dim, e_off, total):
        wire = np.ascontiguousarray(wire, dtype=np.uint8)
        e_bits = np.ascontiguousarray(e_bits, dtype=np.int32)
        e_dim = np.ascontiguousarray(e_dim, dtype=np.uint64)
        e_off = np.ascontiguousarray(e_off, dtype=np.uint64)
        n = len(e_bits)
        ld = int(e_dim.max()) if n else 1
        out = np.zeros((max(1, n), ld), np.float64)
        st = self.L.qo_decode_message_set(_p(wire), len(wire), _p(e_bits), _p(e_dim), _p(e_off),
                                          n, total, _p(out), ld)
        if st:
            raise ValueError(f"decode_message_set: status {st}")
        return out[:n]

    # tensor ops ----------------------------------------------------------
    def aggregate_rows(self, v, h, h_remote, rows, out):
        h = np.ascontiguousarray(h, np.float64)
        d = h.shape[1]
        hr = np.ascontiguousarray(h_remote, np.float64) if h_remote is not None else None
        rows = np.ascontiguousarray(rows, np.int32)
        self.L.qo_aggregate_rows(_p(v["self_alpha"]), _p(v["local_ptr"]), _p(v["local_row"]),
                                 _p(v["local_alpha_fwd"]), _p(v["remote_ptr"]),
                                 _p(v["remote_slot"]), _p(v["remote_alpha"]), _p(h), _p(hr), d,
                                 _p(rows), len(rows), _p(out))
        return out

    def backward_remote_partials(self, v, gbar, num_remote):
        gbar = np.ascontiguousarray(gbar, np.float64)
        d = gbar.shape[1]
        out = np.zeros((num_remote, d), np.float64)
        m = np.ascontiguousarray(v["marginal"], np.int32)
        self.L.qo_backward_remote_partials(_p(v["remote_ptr"]), _p(v["remote_slot"]),
                                           _p(v["remote_alpha"]), _p(m), len(m), _p(gbar), d,
                                           _p(out))
        return out

    def layer_forward_rows(self, h_agg, w, rows, relu, out):
        h_agg = np.ascontiguousarray(h_agg, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        rows = np.ascontiguousarray(rows, np.int32)
        self.L.qo_layer_forward_rows(_p(h_agg), _p(w), w.shape[0], w.shape[1], _p(rows),
                                     len(rows), int(relu), None, _p(out))
        return out

    def input_grad_rows(self, dz, w, rows, out):
        dz = np.ascontiguousarray(dz, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        rows = np.ascontiguousarray(rows, np.int32)
        self.L.qo_input_grad_rows(_p(dz), _p(w), w.shape[0], w.shape[1], _p(rows), len(rows),
                                  _p(out))
        return out

    def matmul_transa(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros((a.shape[1], b.shape[1]), np.float64)
        self.L.qo_matmul_transa(_p(a), _p(b), a.shape[0], a.shape[1], b.shape[1], _p(out))
        return out

    def masked_ce_partial(self, logits, labels, rows, inv_denom):
        logits = np.ascontiguousarray(logits, np.float64)
        labels = np.ascontiguousarray(labels, np.int32)
        rows = np.ascontiguousarray(rows, np.int32)
        grad = np.zeros_like(logits)
        loss = self.L.qo_masked_ce_partial(_p(logits), logits.shape[1], _p(labels), _p(rows),
                                           len(rows), inv_denom, _p(grad))
        return loss, grad

    def adam_step(self, p, m, v, g, t, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
        self.L.qo_adam_step(_p(p), _p(m), _p(v), _p(g), p.size, t, lr, b1, b2, eps)

    def compute_coeffs(self, adj_ptr, adj, sage=False):
        adj_ptr = np.ascontiguousarray(adj_ptr, np.int64)
        adj = np.ascontiguousarray(adj, np.int32)
        n = len(adj_ptr) - 1
        alpha = np.zeros(len(adj), np.float64)
        sa = np.zeros(n, np.float64)
        self.L.qo_compute_coeffs(_p(adj_ptr), _p(adj), n, int(sage), _p(alpha), _p(sa))
        return alpha, sa


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Ref:
    """The reference headers compiled via ref_shim.cpp (oracle/_ref/libqgnn_ref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate_dataset.restype = C.c_void_p
        L.ref_generate_dataset.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_double, C.c_double, C.c_uint64, C.c_double,
                                           C.c_double, C.c_uint64]
        L.ref_dataset_from_arrays.restype = C.c_void_p
        L.ref_dataset_from_arrays.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                              C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p]
        L.ref_dataset_free.argtypes = [C.c_void_p]
        L.ref_dataset_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_dataset_load.restype = C.c_void_p
        L.ref_dataset_load.argtypes = [C.c_char_p]
        L.ref_dataset_sizes.argtypes = [C.c_void_p] * 4
        L.ref_dataset_export.argtypes = [C.c_void_p] * 8
        L.ref_view_build.restype = C.c_void_p
        L.ref_view_build.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                     C.c_uint32, C.c_int]
        L.ref_view_free.argtypes = [C.c_void_p]
        L.ref_view_counts.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_view_export.argtypes = [C.c_void_p] * 15
        L.ref_view_remote_lists.argtypes = [C.c_void_p, C.c_uint64] + [C.c_void_p] * 4
        L.ref_engine_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                     C.c_double]

    def _chk(self, st):
        if st:
            raise RefError(st, self.L.ref_last_error().decode())

    def rng_draws(self, seed, coords, n):
        c = np.array(coords, np.uint64)
        out = np.zeros(n, np.uint64)
        self._chk(self.L.ref_rng_draws(_u64(seed), _p(c), len(c), C.c_uint64(n), _p(out)))
        return out

    def rng_gaussians(self, seed, coords, n):
        c = np.array(coords, np.uint64)
        out = np.zeros(n, np.float64)
        self._chk(self.L.ref_rng_gaussians(_u64(seed), _p(c), len(c), C.c_uint64(n), _p(out)))
        return out

    def quantize(self, h, b, seed, coords):
        h = np.ascontiguousarray(h, np.float64)
        c = np.array(coords, np.uint64)
        nb = (len(h) * b + 7) // 8
        out = np.zeros(max(1, nb), np.uint8)
        s, z = C.c_double(), C.c_double()
        self._chk(self.L.ref_quantize(_p(h), C.c_uint64(len(h)), C.c_int(b), _u64(seed), _p(c),
                                      C.c_int(len(c)), C.byref(s), C.byref(z), _p(out)))
        return s.value, z.value, out[:nb]

    def pack(self, codes, b):
        codes = np.ascontiguousarray(codes, np.uint32)
        nb = (len(codes) * b + 7) // 8
        out = np.zeros(max(1, nb), np.uint8)
        self._chk(self.L.ref_pack(_p(codes), C.c_uint64(len(codes)), C.c_int(b), _p(out)))
        return out[:nb]

    def encode_message_set(self, values, rows, ids, bits, seed, coords):
        values = np.ascontiguousarray(values, np.float64)
        rows = np.ascontiguousarray(rows, np.int64)
        ids = np.ascontiguousarray(ids, np.uint32)
        bits = np.ascontiguousarray(bits, np.int32)
        n, dim = len(ids), values.shape[1]
        cap = sum(25 + (dim * int(b) + 7) // 8 for b in bits)
        out = np.zeros(max(1, cap), np.uint8)
        nbytes = C.c_uint64()
        e_id = np.zeros(max(1, n), np.uint32)
        e_bits = np.zeros(max(1, n), np.int32)
        e_off = np.zeros(max(1, n), np.uint64)
        e_dim = np.zeros(max(1, n), np.uint64)
        c = np.array(coords, np.uint64)
        self._chk(self.L.ref_encode_message_set(
            _p(values), C.c_uint64(values.shape[1]), _p(rows), _p(ids), _p(bits), C.c_uint64(n),
            C.c_uint64(dim), _u64(seed), _p(c), C.c_int(len(c)), _p(out), C.byref(nbytes),
            _p(e_id), _p(e_bits), _p(e_off), _p(e_dim)))
        return out[: nbytes.value], dict(id=e_id[:n], bits=e_bits[:n], off=e_off[:n],
                                         dim=e_dim[:n])

    def decode_message_set(self, wire, index, total):
        wire = np.ascontiguousarray(wire, np.uint8)
        n = len(index["id"])
        ld = int(index["dim"].max()) if n else 1
        out = np.zeros((max(1, n), ld), np.float64)
        self._chk(self.L.ref_decode_message_set(
            _p(wire), C.c_uint64(len(wire)), _p(np.ascontiguousarray(index["id"], np.uint32)),
            _p(np.ascontiguousarray(index["bits"], np.int32)),
            _p(np.ascontiguousarray(index["off"], np.uint64)),
            _p(np.ascontiguousarray(index["dim"], np.uint64)), C.c_uint64(n), C.c_uint64(total),
            _p(out), C.c_uint64(ld)))
        return out[:n]

    # datasets ---------------------------------------------------------------
    def _export(self, h):
        nodes, nnz, fdim = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.L.ref_dataset_sizes(h, C.byref(nodes), C.byref(nnz), C.byref(fdim))
        n, e, f = nodes.value, nnz.value, fdim.value
        g = dict(adj_ptr=np.zeros(n + 1, np.int64), adj=np.zeros(max(1, e), np.int32),
                 features=np.zeros((n, f), np.float64), labels=np.zeros(n, np.int32),
                 train=np.zeros(n, np.uint8), val=np.zeros(n, np.uint8), test=np.zeros(n, np.uint8))
        self.L.ref_dataset_export(h, _p(g["adj_ptr"]), _p(g["adj"]), _p(g["features"]),
                                  _p(g["labels"]), _p(g["train"]), _p(g["val"]), _p(g["test"]))
        g["adj"] = g["adj"][:e]
        return g

    def generate_dataset(self, kind="sbm", nodes=1000, classes=4, feature_dim=32, p_intra=0.01,
                         p_inter=0.001, attach_edges=4, same_class_bias=0.8, sep=1.0, seed=1):
        h = self.L.ref_generate_dataset(1 if kind == "cite" else 0, nodes, classes, feature_dim,
                                        p_intra, p_inter, attach_edges, same_class_bias, sep, seed)
        if not h:
            raise RefError(1, self.L.ref_last_error().decode())
        try:
            return self._export(h)
        finally:
            self.L.ref_dataset_free(h)

    def generate_and_save(self, dir, kind="sbm", nodes=1000, classes=4, feature_dim=32,
                          p_intra=0.01, p_inter=0.001, attach_edges=4, same_class_bias=0.8,
                          sep=1.0, seed=1):
        """generate_dataset then the reference's save_dataset (cli/synth.hpp:153-182)."""
        h = self.L.ref_generate_dataset(1 if kind == "cite" else 0, nodes, classes, feature_dim,
                                        p_intra, p_inter, attach_edges, same_class_bias, sep, seed)
        if not h:
            raise RefError(1, self.L.ref_last_error().decode())
        try:
            self._chk(self.L.ref_dataset_save(h, str(dir).encode()))
            return self._export(h)
        finally:
            self.L.ref_dataset_free(h)

    def load_dataset(self, dir):
        """The reference's load_dataset (cli/synth.hpp:184-205) as arrays."""
        h = self.L.ref_dataset_load(str(dir).encode())
        if not h:
            raise RefError(1, self.L.ref_last_error().decode())
        try:
            return self._export(h)
        finally:
            self.L.ref_dataset_free(h)

    def partition_owner(self, adj_ptr, adj, n_parts, seed):
        n = len(adj_ptr) - 1
        owner = np.zeros(n, np.uint32)
        self._chk(self.L.ref_partition_owner(_p(adj_ptr), _p(adj), C.c_uint64(n),
                                             C.c_uint64(n_parts), _u64(seed), _p(owner)))
        return owner

    def compute_coeffs(self, adj_ptr, adj, sage=False):
        n = len(adj_ptr) - 1
        alpha = np.zeros(len(adj), np.float64)
        sa = np.zeros(n, np.float64)
        self._chk(self.L.ref_compute_coeffs(_p(adj_ptr), _p(adj), C.c_uint64(n), C.c_int(sage),
                                            _p(alpha), _p(sa)))
        return alpha, sa

    def view(self, adj_ptr, adj, owner, n_parts, dev, sage=False):
        return RefView(self, adj_ptr, adj, owner, n_parts, dev, sage)

    # dense ------------------------------------------------------------------
    def layer_forward_rows(self, h_agg, w, rows, relu, out):
        h_agg = np.ascontiguousarray(h_agg, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        rows = np.ascontiguousarray(rows, np.uint32)
        self._chk(self.L.ref_layer_forward_rows(
            _p(h_agg), C.c_uint64(h_agg.shape[0]), _p(w), C.c_uint64(w.shape[0]),
            C.c_uint64(w.shape[1]), C.c_int(int(relu)), _p(rows), C.c_uint64(len(rows)), _p(out)))
        return out

    def input_grad_rows(self, dz, w, rows, out):
        dz = np.ascontiguousarray(dz, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        rows = np.ascontiguousarray(rows, np.uint32)
        self._chk(self.L.ref_input_grad_rows(
            _p(dz), C.c_uint64(dz.shape[0]), _p(w), C.c_uint64(w.shape[0]), C.c_uint64(w.shape[1]),
            _p(rows), C.c_uint64(len(rows)), _p(out)))
        return out

    def matmul_transa(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros((a.shape[1], b.shape[1]), np.float64)
        self._chk(self.L.ref_matmul_transa(_p(a), _p(b), C.c_uint64(a.shape[0]),
                                           C.c_uint64(a.shape[1]), C.c_uint64(b.shape[1]),
                                           _p(out)))
        return out

    def model_init(self, dims, seed):
        d = np.array(dims, np.uint64)
        total = sum(int(dims[i]) * int(dims[i + 1]) for i in range(len(dims) - 1))
        out = np.zeros(total, np.float64)
        self._chk(self.L.ref_model_init(_p(d), C.c_int(len(d)), _u64(seed), _p(out)))
        ws, o = [], 0
        for i in range(len(dims) - 1):
            k = int(dims[i]) * int(dims[i + 1])
            ws.append(out[o: o + k].reshape(int(dims[i]), int(dims[i + 1])))
            o += k
        return ws

    # assigner ---------------------------------------------------------------
    def solve_instance(self, pairs, n_devices, theta, gamma, lam, group_size, brute=False):
        """pairs: list of (src, dst, [(id, dim, lo, hi, asq), ...]).  Returns (bits list, eval)."""
        src = np.array([p[0] for p in pairs], np.uint32)
        dst = np.array([p[1] for p in pairs], np.uint32)
        cnt = np.array([len(p[2]) for p in pairs], np.uint64)
        msgs = [m for p in pairs for m in p[2]]
        mid = np.array([m[0] for m in msgs], np.uint32)
        mdim = np.array([m[1] for m in msgs], np.uint64)
        mlo = np.array([m[2] for m in msgs], np.float64)
        mhi = np.array([m[3] for m in msgs], np.float64)
        masq = np.array([m[4] for m in msgs], np.float64)
        th = np.ascontiguousarray(theta, np.float64)
        ga = np.ascontiguousarray(gamma, np.float64)
        bits = np.zeros(max(1, len(msgs)), np.int32)
        ev = np.zeros(3, np.float64)
        self._chk(self.L.ref_solve_instance(
            C.c_uint64(len(pairs)), _p(src), _p(dst), _p(cnt), _p(mid), _p(mdim), _p(mlo),
            _p(mhi), _p(masq), C.c_uint64(n_devices), _p(th), _p(ga), C.c_double(lam),
            C.c_uint64(group_size), C.c_int(int(brute)), _p(bits), _p(ev)))
        return bits[: len(msgs)], ev

    # engine -----------------------------------------------------------------
    def engine_run(self, g, dims, n_parts, bit_mode=1, fixed_bits=8, epochs=3, seed=7,
                   sage=False, lam=0.5, group_size=4, period=50, threads=False, theta=3e-9,
                   gamma=5e-5, lr=0.01, owner=None, times=None, layer_norm=False, dropout=0.0):
        """Reference Engine::run.  owner: planted owner map -> the Engine
        partitions with partitions_from_owner (else partition_graph, BFS).
        times: optional float64[2] <- (setup seconds, run seconds)."""
        h = self.L.ref_dataset_from_arrays(
            _p(g["adj_ptr"]), _p(g["adj"]), C.c_uint64(len(g["adj_ptr"]) - 1),
            _p(np.ascontiguousarray(g["features"], np.float64)),
            C.c_uint64(g["features"].shape[1]), _p(g["labels"]), _p(g["train"]), _p(g["val"]),
            _p(g["test"]))
        try:
            d = np.array(dims, np.uint64)
            ep = np.zeros((epochs, 10), np.float64)
            total = sum(int(dims[i]) * int(dims[i + 1]) for i in range(len(dims) - 1))
            fw = np.zeros(total, np.float64)
            own = None if owner is None else np.ascontiguousarray(owner, np.uint32)
            self._chk(self.L.ref_engine_run(h, _p(d), len(d), int(sage), int(bit_mode),
                                            int(fixed_bits), lam, group_size, period, epochs,
                                            seed, n_parts, int(threads), theta, gamma, lr,
                                            _p(ep), _p(fw),
                                            _p(own), _p(times), int(layer_norm), float(dropout)))
            return ep, fw
        finally:
            self.L.ref_dataset_free(h)


class RefView:
    """Partition + DeviceAggView of one device under an owner map (aggregate.hpp:41-89)."""

    def __init__(self, ref, adj_ptr, adj, owner, n_parts, dev, sage):
        self.ref = ref
        self.adj_ptr = np.ascontiguousarray(adj_ptr, np.int64)
        self.adj = np.ascontiguousarray(adj, np.int32)
        self.owner = np.ascontiguousarray(owner, np.uint32)
        L = ref.L
        self.h = L.ref_view_build(_p(self.adj_ptr), _p(self.adj), len(self.adj_ptr) - 1,
                                  _p(self.owner), n_parts, dev, int(sage))
        if not self.h:
            raise RefError(1, L.ref_last_error().decode())
        c = np.zeros(6, np.uint64)
        L.ref_view_counts(self.h, _p(c))
        no, nr, ln, rn, nc, nm = (int(x) for x in c)
        self.num_owned, self.num_remote = no, nr
        v = dict(self_alpha=np.zeros(no), local_ptr=np.zeros(no + 1, np.int64),
                 local_row=np.zeros(max(1, ln), np.int32), local_alpha_fwd=np.zeros(max(1, ln)),
                 local_alpha_bwd=np.zeros(max(1, ln)), remote_ptr=np.zeros(no + 1, np.int64),
                 remote_slot=np.zeros(max(1, rn), np.int32), remote_alpha=np.zeros(max(1, rn)),
                 slot_node=np.zeros(max(1, nr), np.uint32),
                 slot_owner=np.zeros(max(1, nr), np.uint32),
                 device_slot_offset=np.zeros(n_parts + 1, np.int64),
                 central=np.zeros(max(1, nc), np.int32), marginal=np.zeros(max(1, nm), np.int32),
                 owned=np.zeros(max(1, no), np.uint32))
        L.ref_view_export(self.h, *[_p(v[k]) for k in (
            "self_alpha", "local_ptr", "local_row", "local_alpha_fwd", "local_alpha_bwd",
            "remote_ptr", "remote_slot", "remote_alpha", "slot_node", "slot_owner",
            "device_slot_offset", "central", "marginal", "owned")])
        for k, n in (("local_row", ln), ("local_alpha_fwd", ln), ("local_alpha_bwd", ln),
                     ("remote_slot", rn), ("remote_alpha", rn), ("slot_node", nr),
                     ("slot_owner", nr), ("central", nc), ("marginal", nm), ("owned", no)):
            v[k] = v[k][:n]
        ins = np.zeros(n_parts, np.uint64)
        outs = np.zeros(n_parts, np.uint64)
        L.ref_view_remote_lists(self.h, n_parts, _p(ins), _p(outs), None, None)
        in_ids = np.zeros(max(1, int(ins.sum())), np.uint32)
        out_ids = np.zeros(max(1, int(outs.sum())), np.uint32)
        L.ref_view_remote_lists(self.h, n_parts, _p(ins), _p(outs), _p(in_ids), _p(out_ids))
        io, oo = np.concatenate([[0], np.cumsum(ins)]), np.concatenate([[0], np.cumsum(outs)])
        v["remote_in"] = [in_ids[int(io[q]): int(io[q + 1])] for q in range(n_parts)]
        v["remote_out"] = [out_ids[int(oo[q]): int(oo[q + 1])] for q in range(n_parts)]
        self.v = v

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_view_free(self.h)
            self.h = None

    def aggregate_rows(self, h, h_remote, rows, out):
        h = np.ascontiguousarray(h, np.float64)
        hr = np.ascontiguousarray(h_remote, np.float64) if h_remote is not None else None
        rows = np.ascontiguousarray(rows, np.uint32)
        self.ref._chk(self.ref.L.ref_view_aggregate_rows(
            self.h, _p(h), _p(hr), C.c_uint64(h.shape[1]), _p(rows), C.c_uint64(len(rows)),
            _p(out)))
        return out

    def aggregate_backward_local(self, gbar, rows, out):
        gbar = np.ascontiguousarray(gbar, np.float64)
        rows = np.ascontiguousarray(rows, np.uint32)
        self.ref._chk(self.ref.L.ref_view_aggregate_backward_local(
            self.h, _p(gbar), C.c_uint64(gbar.shape[1]), _p(rows), C.c_uint64(len(rows)),
            _p(out)))
        return out

    def backward_remote_partials(self, gbar):
        gbar = np.ascontiguousarray(gbar, np.float64)
        out = np.zeros((self.num_remote, gbar.shape[1]), np.float64)
        self.ref._chk(self.ref.L.ref_view_backward_remote_partials(
            self.h, _p(gbar), C.c_uint64(gbar.shape[1]), _p(out)))
        return out


port = _Port()


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class _LazyRef:
    _inst = None

    def __getattr__(self, name):
        if _LazyRef._inst is None:
            _LazyRef._inst = _Ref()
        return getattr(_LazyRef._inst, name)


ref = _LazyRef()
