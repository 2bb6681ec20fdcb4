"""Generate golden fixtures from the reference itself (oracle/_ref/libqgnn_ref.so).

Run in the dev container (needs the compiled reference):  python tests/golden/make_golden.py
Outputs tests/golden/golden.npz.  Every vector is produced by the UNMODIFIED
reference headers (quant.hpp, codec.hpp, aggregate.hpp, model.hpp,
partition.hpp, solve.hpp, engine.hpp) through oracle/ref_shim.cpp.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402


def main():
    g = {}
    rs = np.random.default_rng(20240901)
    # --- quantize: rows of various dims/widths, incl. constant + post-relu rows
    dims = [1, 5, 37, 100, 128, 256, 602]
    qi = 0
    for d in dims:
        for b in (2, 4, 8):
            for kind in ("gauss", "relu", "const"):
                h = rs.standard_normal(d) * 2.0
                if kind == "relu":
                    h = np.maximum(h, 0.0)
                if kind == "const":
                    h = np.full(d, 0.75)
                coords = [2, 1 + qi % 3, qi % 5, 0, 1, 1000 + qi]
                s, z, p = ref.quantize(h, b, 7, coords)
                g[f"q{qi}_h"] = h
                g[f"q{qi}_meta"] = np.array([b, 7] + coords, np.uint64)
                g[f"q{qi}_sz"] = np.array([s, z])
                g[f"q{qi}_payload"] = p
                qi += 1
    g["n_quant"] = np.array(qi)
    # --- encode_message_set: 40 messages, mixed widths, f32-representable values
    vals = rs.standard_normal((50, 96)).astype(np.float32).astype(np.float64)
    rows = rs.permutation(50)[:40].astype(np.int64)
    ids = (rs.permutation(10000)[:40] * 7 + 3).astype(np.uint32)
    bits = rs.choice([2, 4, 8], 40).astype(np.int32)
    coords = [2, 3, 1, 0, 1]
    wire, idx = ref.encode_message_set(vals, rows, ids, bits, 11, coords)
    g.update(enc_vals=vals, enc_rows=rows, enc_ids=ids, enc_bits=bits,
             enc_coords=np.array([11] + coords, np.uint64), enc_wire=wire, enc_idx_id=idx["id"],
             enc_idx_bits=idx["bits"], enc_idx_off=idx["off"], enc_idx_dim=idx["dim"])
    dec = ref.decode_message_set(wire, idx, len(wire))
    g["enc_decoded"] = dec
    # --- graph: reference SBM generator, BFS partition, views, aggregation
    ds = ref.generate_dataset("sbm", nodes=120, classes=3, feature_dim=8, p_intra=0.08,
                              p_inter=0.008, sep=1.5, seed=5)
    for k in ("adj_ptr", "adj", "features", "labels", "train", "val", "test"):
        g[f"g_{k}"] = ds[k]
    owner = ref.partition_owner(ds["adj_ptr"], ds["adj"], 4, 11)
    g["g_owner_p4_s11"] = owner
    alpha, sa = ref.compute_coeffs(ds["adj_ptr"], ds["adj"], sage=False)
    g["g_alpha_gcn"], g["g_self_alpha"] = alpha, sa
    alpha_s, _ = ref.compute_coeffs(ds["adj_ptr"], ds["adj"], sage=True)
    g["g_alpha_sage"] = alpha_s
    v = ref.view(ds["adj_ptr"], ds["adj"], owner, 4, 1)
    h = rs.standard_normal((v.num_owned, 8))
    hr = rs.standard_normal((v.num_remote, 8))
    out = np.zeros((v.num_owned, 8))
    rows_all = np.arange(v.num_owned, dtype=np.uint32)
    v.aggregate_rows(h, hr, rows_all, out)
    g.update(agg_h=h, agg_hr=hr, agg_out=out)
    gb = rs.standard_normal((v.num_owned, 8))
    g["agg_gbar"] = gb
    g["agg_partials"] = v.backward_remote_partials(gb)
    ob = np.zeros((v.num_owned, 8))
    v.aggregate_backward_local(gb, rows_all, ob)
    g["agg_bwd_local"] = ob
    # --- dense
    w = ref.model_init([8, 12, 3], 11)
    g["w0"], g["w1"] = w[0], w[1]
    fo = np.zeros((v.num_owned, 12))
    ref.layer_forward_rows(h, w[0], rows_all, True, fo)
    g["dense_fwd"] = fo
    dz = rs.standard_normal((v.num_owned, 12))
    ig = np.zeros((v.num_owned, 8))
    ref.input_grad_rows(dz, w[0], rows_all, ig)
    g.update(dense_dz=dz, dense_igrad=ig, dense_wgrad=ref.matmul_transa(h, dz))
    # --- engine: losses of the reference trainer (test_trainer.cpp settings)
    for mode, fb, name in ((0, 8, "fp"), (1, 8, "f8"), (1, 2, "f2"), (2, 8, "uni")):
        ep, fw = ref.engine_run(ds, [8, 12, 3], 4, bit_mode=mode, fixed_bits=fb, epochs=5,
                                seed=11, period=5)
        g[f"eng_{name}_epochs"] = ep
        g[f"eng_{name}_weights"] = fw
    ep, fw = ref.engine_run(ds, [8, 12, 3], 4, bit_mode=3, epochs=12, seed=11, period=5,
                            group_size=4, theta=3e-9, gamma=5e-5)
    g["eng_ad_epochs"], g["eng_ad_weights"] = ep, fw
    # GraphSAGE-mean aggregation (coeffs.hpp kSageMean) and a 3-layer GCN
    ep, fw = ref.engine_run(ds, [8, 12, 3], 4, bit_mode=1, fixed_bits=8, epochs=5, seed=11,
                            period=5, sage=True)
    g["eng_sage_epochs"], g["eng_sage_weights"] = ep, fw
    ep, fw = ref.engine_run(ds, [8, 16, 16, 3], 4, bit_mode=1, fixed_bits=4, epochs=5, seed=11,
                            period=5)
    g["eng_l3_epochs"], g["eng_l3_weights"] = ep, fw
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print("wrote", os.path.join(HERE, "golden.npz"), len(g), "arrays")


if __name__ == "__main__":
    main()
