"""Generate tests/golden/ref_golden.npz from the PRISTINE reference (oracle/_ref).

Run in a container where /root/reference exists:  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs /root/reference.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

O.build(ref=True)
R = O.Ref()
G = {}
meta = {"generator": "tests/golden/make_golden.py", "source": "pristine reference oracle/_ref"}

# Philox4x32-10 known answers (Random123's published KAT vectors) through the reference
kat = [((0, 0), (0, 0, 0, 0)),
       ((0xa4093822, 0x299f31d0), (0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344)),
       ((0xffffffff, 0xffffffff), (0xffffffff, 0xffffffff, 0xffffffff, 0xffffffff))]
G["philox_in"] = np.array([list(k) + list(c) for k, c in kat], dtype=np.uint64)
G["philox_out"] = np.array([R.philox(k, c) for k, c in kat], dtype=np.uint64)
G["normals_1_0_0"] = R.normals(1, 0, 0, 16)
G["normals_7_3_big"] = R.normals(7, 3, (1 << 33) + 5, 16)

# spectra: SPEC examples + a padded Matérn case
cases = {"sepexp_m2_l1": (2, O.SEP_EXP, 1.0, 1.0, 1.0), "sepexp_m8_l01": (8, O.SEP_EXP, 1.0, 0.1, 1.0),
         "matern_m8_nu05": (8, O.MATERN, 1.0, 0.1, 0.5), "matern_m16_nu15_pad": (16, O.MATERN, 1.0, 0.3, 1.5),
         "matern_m16_nu15": (16, O.MATERN, 2.0, 0.05, 1.5)}
for name, (m, fam, s2, lam, nu) in cases.items():
    op = R.build_operator(m, fam, s2, lam, nu)
    G[f"eig_{name}"] = op.eigenvalues()
    G[f"J_{name}"] = np.array([op.J])
    G[f"perm_{name}"] = op.perm()

# CE sample + restriction: m = 16 Matérn ν=1.5 λ=0.05, ξ = NormalStream(1, 0, i), i < 3
op = R.build_operator(16, O.MATERN, 2.0, 0.05, 1.5)
xi = np.stack([R.normals(1, 0, i, op.s) for i in range(3)])
G["ce_xi"] = xi
G["ce_fine"] = np.stack([op.restrict(op.sample(x), 16) for x in xi])
G["ce_coarse"] = np.stack([op.restrict(op.sample(x), 8) for x in xi])
tr = op.truncated(op.s // 2)
G["ce_fine_trunc"] = np.stack([tr.restrict(tr.sample(x), 16) for x in xi])

# FEM: solve the m=16 fields, flow-cell, f=1, MG, tol 1e-10
G["fem_u"] = np.stack([R.solve(16, z) for z in G["ce_fine"]])
G["fem_qpoint"] = np.array([R.qoi_point(16, u) for u in G["fem_u"]])
G["fem_ql2"] = np.array([R.qoi_l2(16, u) for u in G["fem_u"]])

# coupled samples on a level (h0 = 1/8, ℓ = 1 → m = 16 / 8), sep-exp λ=0.1, point QoI
opts = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=0.1, nu_or_p=1.0, seed=1)
plan = R.plan(1, 1.0 / 8, opts)
qf, qc, _ = R.coupled(plan, True, False, False, opts, 0, 6)
G["coupled_qf"], G["coupled_qc"] = qf, qc
# smoothed level (HalfSpectrum): finest CES level pairs untruncated fine with truncated coarse
opts_s = O.RefOpts.make(family=O.SEP_EXP, sigma2=1.0, lam=0.1, nu_or_p=1.0, seed=1, smoothing=1)
plan_s = R.plan(1, 1.0 / 8, opts_s)
G["coupled_s_k"] = np.array([plan_s.k_trunc])
G["coupled_s_eig"] = plan_s.op().eigenvalues()
qf, qc, _ = R.coupled(plan_s, True, False, True, opts_s, 0, 6)
G["coupled_s_qf"], G["coupled_s_qc"] = qf, qc

# single-level MC estimate (config-1 analogue, small): m = 16, N = 64, L2 QoI
opts_mc = O.RefOpts.make(family=O.MATERN, sigma2=1.0, lam=0.1, nu_or_p=0.5, qoi_kind=1, seed=1)
rep = R.mc_fixed_n(opts_mc, 16, 64)
G["mc16_mean_var"] = np.array([rep.levels()[0]["mean_y"], rep.levels()[0]["var_y"]])

# estimator host math
G["k_ell"] = np.array([R.choose_k_ell(O.SEP_EXP, 1.0, 0.01, 1.0, h, 0, int((2 / h) ** 2))
                       for h in (1 / 16, 1 / 32, 1 / 64)]
                      + [R.choose_k_ell(O.MATERN, 1.0, 0.1, 1.5, h, 0, int((2 / h) ** 2))
                         for h in (1 / 16, 1 / 32)])
G["coarsest_bound"] = np.array([R.coarsest_level_bound(O.SEP_EXP, 1, 0.01, 1),
                                R.coarsest_level_bound(O.MATERN, 1, 0.03, 1.5)])

np.savez_compressed(os.path.join(os.path.dirname(__file__), "ref_golden.npz"), **G)
with open(os.path.join(os.path.dirname(__file__), "ref_golden.json"), "w") as f:
    json.dump(meta | {"keys": sorted(G)}, f, indent=1)
print("wrote", len(G), "arrays")
