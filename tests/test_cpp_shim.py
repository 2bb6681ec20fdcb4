"""The reference-side C++ binding (include/qgnn_b200_shim.hpp) compiled against
the unmodified reference headers (tests/cpp/Makefile) and checked against the
reference's own operators: partitions_from_owner, DeviceAggView::build,
Lookup::bits_for on the host; encode/decode_message_set, aggregate_rows,
aggregate_backward_local, backward_remote_partials, layer_forward_rows,
input_grad_rows and matmul_transa on the GPU (bit for bit, same exceptions)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
BIN = os.path.join(CPP, "_build", "shim_parity")


def _binary():
    if os.path.isdir("/root/reference/proj/include/qgnn"):
        subprocess.run(["make", "-s", "-C", CPP], check=True, capture_output=True)
    if not os.path.exists(BIN):
        pytest.skip("shim_parity not built (needs the reference headers at build time)")
    return BIN


def test_cpp_shim_host_operators_match_reference():
    r = subprocess.run([_binary(), "--host"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_shim_device_operators_match_reference(cuda):
    r = subprocess.run([_binary(), "--all"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
