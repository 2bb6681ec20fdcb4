"""§8f rank 1 at N = 1: the forward marginal SpMM reads the halo rows straight from
the exchange arena (8/4/2-bit chunks dequantized in registers, K3 and the fp32
halo gone for the aggregate-first layers).  The dequantized values are K3's
(fmaf(code, S, Z)) and the accumulation order is unchanged, so every epoch's
loss/accuracy and the final weights must be bit-identical to the K3 path."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HELPER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "engine_digest.py")


def _digest(env, *args):
    out = subprocess.run([sys.executable, HELPER, *args], capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=900, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


@pytest.mark.parametrize("mode,bits", [("adaptive", "8"), ("fixed", "4"), ("fixed", "2"),
                                       ("fp", "8")])
def test_packed_halo_bit_identical_to_k3_path(cuda, mode, bits):
    ref = _digest({"QGNN_PACKED_HALO": "0"}, mode, bits)
    got = _digest({"QGNN_PACKED_HALO": "1"}, mode, bits)
    assert got["epochs"] == ref["epochs"]
    assert got["weights_sha"] == ref["weights_sha"]
    # K3 forward launches gone for the two aggregate-first layers (8 partitions each)
    assert ref["dequant_launches"] - got["dequant_launches"] == 4 * 2 * 8
