"""Pin the CPU oracle (oracle/osc_oracle.c) against the reference's golden vectors (tests/golden,
generated from the pristine reference by tests/golden/make_golden.py) and, where available,
against the pristine reference itself (oracle/_ref)."""
import numpy as np
import pytest


def test_philox_kat(port, golden):
    for row, out in zip(golden["philox_in"], golden["philox_out"]):
        assert port.philox(tuple(int(x) for x in row[:2]), tuple(int(x) for x in row[2:])) == \
            [int(x) for x in out]
    # Random123 published KAT for philox4x32_10(ctr=0, key=0)
    assert [int(x) for x in golden["philox_out"][0]] == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]


def test_normals(port, golden):
    assert np.array_equal(port.normals(1, 0, 0, 16), golden["normals_1_0_0"])
    assert np.array_equal(port.normals(7, 3, (1 << 33) + 5, 16), golden["normals_7_3_big"])


def test_sample_and_restrict(port, golden):
    eig = golden["eig_matern_m16_nu15"]
    sl = np.sqrt(np.maximum(eig, 0))
    n = 32
    for b in range(3):
        u = port.sample(n, sl, golden["ce_xi"][b])
        f = port.restrict(n, 16, u, 16)
        c = port.restrict(n, 16, u, 8)
        assert np.max(np.abs(f - golden["ce_fine"][b])) <= 1e-13 * np.max(np.abs(f))
        assert np.max(np.abs(c - golden["ce_coarse"][b])) <= 1e-13 * np.max(np.abs(c))


def test_solve_bit_exact(port, golden):
    for b in range(3):
        u, it, rc, _ = port.solve(16, golden["ce_fine"][b])
        assert rc == 0
        assert np.array_equal(u, golden["fem_u"][b])  # same operation order as fem.cpp
        assert port.qoi(16, u) == golden["fem_qpoint"][b]
        assert port.qoi(16, u, qoi=1) == golden["fem_ql2"][b]


def test_coupled(port, golden):
    from paper_2306_13493_b200 import api  # host setup only (no GPU call)
    op = api.build_operator(api.GridSpec.square(16), api.CovarianceModel.separable_exponential(1, 0.1))
    sl = np.sqrt(np.maximum(op.eigenvalues, 0))
    qf, qc, itf, itc = port.coupled(16, op.n, sl, None, True, 1, 1, 0, 6, threads=2)
    assert np.max(np.abs(qf - golden["coupled_qf"]) / np.abs(golden["coupled_qf"])) < 1e-12
    assert np.max(np.abs(qc - golden["coupled_qc"]) / np.abs(golden["coupled_qc"])) < 1e-12
    assert np.all(itf > 0) and np.all(itc > 0)


def test_moments(port, golden):
    rng = np.random.default_rng(1)
    qf, qc = rng.standard_normal(100), rng.standard_normal(100)
    mo = port.moments(qf, qc, True)
    y = qf - qc
    assert abs(mo["mean_y"] - y.mean()) < 1e-14 and abs(mo["var_y"] - y.var(ddof=1)) < 1e-13


def test_spec_known_answers(port):
    # SPEC fem: Z ≡ 0, f = 0 → u = 1 − x; point QoI 8/15; L2 1/√3; flux 1; ∫u = 1/2
    m = 8
    u, it, rc, _ = port.solve(m, np.zeros((m + 1) ** 2), forcing=0)
    x = np.tile(np.arange(m + 1) / m, m + 1)
    assert np.max(np.abs(u - (1 - x))) < 1e-10
    assert abs(port.qoi(m, u) - 8 / 15) < 1e-10
    assert abs(port.qoi(m, u, qoi=1) - 1 / np.sqrt(3)) < 1e-10
    assert abs(port.qoi(m, u, qoi=2) - 0.5) < 1e-10
    assert abs(port.qoi(m, u, qoi=3, forcing=0) - 1.0) < 1e-10
    # homogeneous Dirichlet, f = 1, k = 1: ∫u ≈ 0.0351 (series solution of −Δu = 1), flux ≈ 0 side share
    u, it, rc, _ = port.solve(64, np.zeros(65 ** 2), bc=1, forcing=1)
    assert rc == 0 and abs(port.qoi(64, u, bc=1, qoi=2) - 0.035144) < 2e-4


def test_port_matches_pristine_reference(port, ref):
    """Only where oracle/_ref exists: solve + sample bit-identity on fresh inputs."""
    op = ref.build_operator(32, 0, 1.0, 0.05, 0.5)
    xi = ref.normals(3, 1, 12, op.s)
    u = op.sample(xi)
    sl = np.sqrt(np.maximum(op.eigenvalues(), 0))
    assert np.max(np.abs(port.sample(op.n, sl, xi) - u)) < 1e-13 * np.max(np.abs(u))
    Z = op.restrict(u, 32)
    uo, it, rc, _ = port.solve(32, Z)
    assert np.array_equal(uo, ref.solve(32, Z))
