"""Full-size parity on the B200: the BASELINE.json configurations at the sizes
they are benchmarked at, checked against independent answers (the CPU oracle
cannot reach 30+ qubits, SURVEY §8c "Limits of the oracle").

* Config 2 (QFT-30 c128, the bench's exact path: lazy |0...0>, NVRTC passes,
  <Z_i> fused into the last pass) against the closed form of the QFT of a
  product state: for psi = (x)_q (c_q|0> + s_q|1>),
      QFT psi [k] = 2^{-n/2} prod_q (c_q + s_q exp(2 pi i (k 2^q mod 2^n) / 2^n)),
  the same DFT convention the reference pins in `test_statevector.py:52-76`.
  Every one of the 2^30 amplitudes and every <Z_i> is compared.
* Config 3 (Sycamore-32 d20 c64): mirror circuit U U^dag |0> = |0>
  (`metrics.py:33-56`), and the c64 state against the c128 state of the same
  circuit (both on the device, compared by svb_compare).
* Capacity: x-prep QFT at 33 qubits c128 and 34 qubits c64 (128 GiB each)
  against the DFT column (`test_statevector.py:52-62`), and GHZ-33.

Closed forms are evaluated with torch in float64 on the GPU, chunk by chunk,
beside the amplitudes read back through the C ABI."""
import math

import numpy as np
import pytest

from paper_2512_04216_b200 import statevector as sv
from paper_2512_04216_b200 import suite
from paper_2512_04216_b200.circuit import Circuit, inverse_circuit

pytestmark = pytest.mark.gpu

CHUNK = 1 << 24


def _torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def _product_qft_chunk(torch, n, cs, ss, off, cnt):
    """QFT of the product state (x)_q (cs[q]|0> + ss[q]|1>) at k in [off, off+cnt)."""
    N = 1 << n
    k = torch.arange(off, off + cnt, dtype=torch.int64, device="cuda")
    acc = torch.ones(cnt, dtype=torch.complex128, device="cuda")
    for q in range(n):
        ph = ((k << q) & (N - 1)).to(torch.float64) * (2 * math.pi / N)
        acc *= torch.complex(cs[q] + ss[q] * torch.cos(ph), ss[q] * torch.sin(ph))
    return acc / math.sqrt(N), k


def _compare_chunks(torch, state, n, cs, ss, offsets, zq=None):
    """(normwise relerr over the given chunks, <Z_q> of the closed form if zq)."""
    err2 = ref2 = 0.0
    z = np.zeros(len(zq or []))
    buf = np.empty(CHUNK, dtype=np.complex128)
    for off in offsets:
        cnt = min(CHUNK, (1 << n) - off)
        want, k = _product_qft_chunk(torch, n, cs, ss, off, cnt)
        got = torch.from_numpy(state.read(off, cnt, buf[:cnt])).to("cuda")
        err2 += float(torch.sum(torch.abs(got - want) ** 2))
        ref2 += float(torch.sum(torch.abs(want) ** 2))
        if zq:
            p = torch.abs(want) ** 2
            for j, q in enumerate(zq):
                sign = 1.0 - 2.0 * ((k >> q) & 1).to(torch.float64)
                z[j] += float(torch.sum(p * sign))
    return math.sqrt(err2 / ref2), z


def test_qft30_bench_path_vs_closed_form():
    """Config 2 exactly as bench.py runs it: DeviceState.zero() + apply_gates_z
    (JIT passes, support tracking, free initial layout, fused <Z_i>), 2^30
    amplitudes at 1e-10 normwise and <Z_i> at 1e-10 absolute."""
    torch = _torch()
    n = 30
    c = suite.qft_bench_circuit(n)
    gates = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, "c128")
    for _ in range(2):  # the second step reuses the cached program, as the bench's timed steps do
        s.zero()
        z = s.apply_gates_z(gates, list(range(n)))
    theta = [0.1 * (q + 1) for q in range(n)]
    cs = [math.cos(t / 2) for t in theta]
    ss = [math.sin(t / 2) for t in theta]
    rel, zref = _compare_chunks(torch, s, n, cs, ss, range(0, 1 << n, CHUNK), zq=list(range(n)))
    assert rel < 1e-10, rel
    np.testing.assert_allclose(z, zref, atol=1e-10)
    np.testing.assert_allclose(s.expect_z([1 << q for q in range(n)]), zref, atol=1e-10)
    s.close()


@pytest.mark.parametrize("n,fused_z", [(24, True), (25, False), (26, True), (27, False), (28, True), (29, False)])
def test_qft_lazy_zero_bulk_row_store_sizes_vs_closed_form(n, fused_z):
    """The bench's program shape at 24..29 qubits: the last pass is the
    one-round direct pass whose tile rows leave as bulk copies (SVB_BULK_ROWS),
    with and without the fused <Z> sums; structure-only (n < 28) and immediate
    (n >= 28) NVRTC bodies.  Amplitudes at 1e-10 normwise, <Z_i> at 1e-10."""
    torch = _torch()
    c = suite.qft_bench_circuit(n)
    gates = sv.gate_array(c.instructions)
    s = sv.DeviceState(n, "c128")
    for _ in range(2):
        s.zero()
        if fused_z:
            z = s.apply_gates_z(gates, list(range(n)))
        else:
            s.apply_gates(gates)
    theta = [0.1 * (q + 1) for q in range(n)]
    cs = [math.cos(t / 2) for t in theta]
    ss = [math.sin(t / 2) for t in theta]
    rel, zref = _compare_chunks(torch, s, n, cs, ss, range(0, 1 << n, CHUNK), zq=list(range(n)))
    assert rel < 1e-10, rel
    if fused_z:
        np.testing.assert_allclose(z, zref, atol=1e-10)
    s.close()


def test_qft30_round_trip_restores_product_state():
    """ry-prep QFT-30 then QFT^-1 (the bench circuit and its inverse, one
    program) returns the analytic product state (x)_q ry(0.1 (q+1))|0>."""
    torch = _torch()
    n = 30
    c = suite.qft_bench_circuit(n)
    body = [i for i in c.instructions if i.kind != "ry"]
    inv = inverse_circuit(Circuit(n, 0, body)).instructions
    s = sv.DeviceState(n, "c128")
    s.apply_instructions(list(c.instructions) + list(inv))
    theta = [0.1 * (q + 1) for q in range(n)]
    err2 = ref2 = 0.0
    buf = np.empty(CHUNK, dtype=np.complex128)
    for off in range(0, 1 << n, CHUNK):
        k = torch.arange(off, off + CHUNK, dtype=torch.int64, device="cuda")
        want = torch.ones(CHUNK, dtype=torch.float64, device="cuda")
        for q in range(n):
            b = ((k >> q) & 1).to(torch.float64)
            want *= math.cos(theta[q] / 2) * (1 - b) + math.sin(theta[q] / 2) * b
        got = torch.from_numpy(s.read(off, CHUNK, buf)).to("cuda")
        err2 += float(torch.sum(torch.abs(got - want) ** 2))
        ref2 += float(torch.sum(want ** 2))
    assert math.sqrt(err2 / ref2) < 1e-10
    s.close()


def test_sycamore32_c64_mirror_and_c128_agreement():
    """Config 3 circuit (4x8 grid, depth 20, seed 0): U U^dag |0> = |0> at c64
    within 1e-5, and the c64 state of U|0> equals the c128 state within 1e-5
    normwise (device-side comparison); fused <Z_i> of both agree."""
    n = 32
    c = suite.sycamore_circuit(4, 8, 20, 0, measured=False)
    inv = inverse_circuit(c)
    m = sv.DeviceState(n, "c64")
    m.apply_instructions(list(c.instructions) + list(inv.instructions))
    a0 = complex(m.read(0, 1)[0])
    norm2 = float(m.expect_z([0])[0])
    dist = math.sqrt(abs(a0 - 1.0) ** 2 + max(norm2 - abs(a0) ** 2, 0.0))
    m.close()
    assert dist < 1e-5, dist
    g = sv.gate_array(c.instructions)
    lo = sv.DeviceState(n, "c64")
    z64 = lo.apply_gates_z(g, list(range(n)))
    hi = sv.DeviceState(n, "c128")
    z128 = hi.apply_gates_z(g, list(range(n)))
    cmp = lo.compare(hi)
    assert cmp["rel"] < 1e-5, cmp
    assert abs(cmp["norm2_other"] - 1.0) < 1e-10
    np.testing.assert_allclose(z64, z128, atol=2e-5)
    lo.close()
    hi.close()


def _dft_capacity(n, precision, tol):
    torch = _torch()
    basis = (0x5A5A5A5A5A >> 3) & ((1 << n) - 1)
    c = Circuit(n)
    for q in range(n):
        if (basis >> q) & 1:
            c.gate("x", q)
    suite.qft(n, c)
    s = sv.DeviceState(n, precision)
    z = s.apply_gates_z(sv.gate_array(c.instructions), list(range(n)))
    assert float(np.max(np.abs(z))) < (1e-10 if precision == "c128" else 2e-5)
    # |basis> is the product state with c_q, s_q in {0, 1}
    cs = [0.0 if (basis >> q) & 1 else 1.0 for q in range(n)]
    ss = [1.0 - x for x in cs]
    N = 1 << n
    offs = [0, N - CHUNK, (N // 3) & ~(CHUNK - 1), (N // 2 + 12345 * CHUNK) % N & ~(CHUNK - 1)]
    rel, _ = _compare_chunks(torch, s, n, cs, ss, offs)
    assert rel < tol, rel
    assert abs(float(s.expect_z([0])[0]) - 1.0) < (1e-10 if precision == "c128" else 1e-5)
    s.close()


def test_capacity_qft33_c128_dft_column():
    _dft_capacity(33, "c128", 1e-10)


def test_capacity_qft34_c64_dft_column():
    _dft_capacity(34, "c64", 1e-5)


def test_capacity_ghz33_c128():
    n = 33
    s = sv.DeviceState(n, "c128")
    s.apply_instructions(suite.ghz_circuit(n, measured=False).instructions)
    r = 1 / math.sqrt(2)
    assert abs(complex(s.read(0, 1)[0]) - r) < 1e-12
    assert abs(complex(s.read((1 << n) - 1, 1)[0]) - r) < 1e-12
    assert abs(float(s.expect_z([0])[0]) - 1.0) < 1e-12
    np.testing.assert_allclose(s.expect_z([1 << q for q in range(n)]), 0.0, atol=1e-12)
    s.close()


_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
from paper_2512_04216_b200 import statevector as sv, suite
n = 28
g = sv.gate_array(suite.qft_bench_circuit(n).instructions)
s = sv.DeviceState(n, "c128")
s.zero()
z = s.apply_gates_z(g, list(range(n)))
buf = np.empty(1 << 20, dtype=np.complex128)
head = s.read(0, 1 << 20, buf).copy()
tail = s.read((1 << n) - (1 << 20), 1 << 20, buf).copy()
np.savez(sys.argv[1], z=z, head=head, tail=tail)
"""


def test_bulk_store_and_product_tree_match_their_plain_variants(tmp_path):
    """The bench-shaped QFT-28 (immediates, product-state round 0, bulk-row
    stores on the last pass) against the same program with register stores
    (SVB_BULK_ROWS=0) and without the product tree (SVB_NO_PROD_FUSE=1), each
    in its own process (the knobs are read once): the stores must agree bit
    for bit, the reassociated arithmetic to 1e-12."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "variant.py"
    script.write_text(_VARIANT_SCRIPT)
    out = {}
    for name, env in (("default", {}), ("regstores", {"SVB_BULK_ROWS": "0"}), ("noprod", {"SVB_NO_PROD_FUSE": "1"})):
        path = tmp_path / f"{name}.npz"
        subprocess.run([sys.executable, str(script), str(path), root], check=True, env={**os.environ, **env},
                       timeout=600)
        out[name] = np.load(path)
    for k in ("z", "head", "tail"):
        np.testing.assert_array_equal(out["default"][k], out["regstores"][k])
        np.testing.assert_allclose(out["default"][k], out["noprod"][k], rtol=0, atol=1e-12)
