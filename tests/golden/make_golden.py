"""Generate golden vectors from the REFERENCE itself (oracle/_ref, i.e.
/root/reference/proj/src compiled unmodified by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/golden.npz; tests compare both the C restatement
(oracle/pirk_oracle.c) and the CUDA path against it.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2001_10635_b200 as pk  # noqa: E402  (model descriptors only)
from oracle import oracle as O  # noqa: E402


def cases():
    out = []
    # config 3 shape at test size: traffic CTMM + GB, stride 10 (configs/traffic.cfg)
    out.append(("traffic_mm_n2000", O.METHOD_MM, pk.make_traffic(2000), 10.0, 20.0, [4.0], [6.0],
                0.0, 30.0, 0.5, 10, {}))
    out.append(("traffic_gb_n2000", O.METHOD_GB, pk.make_traffic(2000), 10.0, 20.0, [4.0], [6.0],
                0.0, 30.0, 0.5, 10, {}))
    # heat3d.cfg verbatim (grid 8, MM, stride 5) and a larger grid
    out.append(("heat_mm_g8", O.METHOD_MM, pk.make_heat3d(8), 0.9, 1.1, None, None, 0.0, 0.05,
                0.002, 5, {}))
    out.append(("heat_gb_g8", O.METHOD_GB, pk.make_heat3d(8), 0.9, 1.1, None, None, 0.0, 0.05,
                0.002, 5, {}))
    out.append(("heat_mm_g24", O.METHOD_MM, pk.make_heat3d(24), 0.9, 1.1, None, None, 0.0, 0.002,
                0.0002, 3, {}))
    # config 4 interpretation at test size
    n = 3000
    c = 2.0 * np.array([O.u01(7, 0, i) for i in range(n)]) - 1.0
    out.append(("chain_mm_n3000", O.METHOD_MM, pk.make_chain(n), c - 0.05, c + 0.05, [-0.1], [0.1],
                0.0, 1.0, 0.01, 10, {}))
    # configs 1/2: arch-quadrotor.cfg (GB as shipped, CTMM via the Jacobian decomposition, MC)
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    aq = pk.make_arch_quadrotor()
    out.append(("archquad_gb", O.METHOD_GB, aq, lo, -lo, None, None, 0.0, 1.0, 0.01, 10, {}))
    out.append(("archquad_mm_jac", O.METHOD_MM, pk.with_jacobian_decomposition(aq), lo, -lo,
                None, None, 0.0, 1.0, 0.01, 10, {}))
    out.append(("archquad_mc_m2000", O.METHOD_MC, aq, lo, -lo, None, None, 0.0, 1.0, 0.01, 10,
                {"samples": 2000, "seed": 1}))
    # laub-loomis.cfg: GB and bit-exact MC
    ll_lo = np.array([1.15, 1.00, 1.45, 2.35, 0.95, 0.05, 0.40])
    ll = pk.make_laub_loomis()
    out.append(("laubloomis_gb", O.METHOD_GB, ll, ll_lo, ll_lo + 0.1, None, None, 0.0, 1.0, 0.005,
                20, {}))
    out.append(("laubloomis_mc_m3000", O.METHOD_MC, ll, ll_lo, ll_lo + 0.1, None, None, 0.0, 1.0,
                0.005, 20, {"samples": 3000, "seed": 1}))
    # test_reach.cpp:88-111 fixture: traffic n=6, seed 42, m=64, stride 2
    out.append(("traffic_mc_n6_seed42", O.METHOD_MC, pk.make_traffic(6), 10.0, 20.0, [4.0], [6.0],
                0.0, 3.0, 0.5, 2, {"samples": 64, "seed": 42}))
    # closed forms (test_reach.cpp:53-75)
    out.append(("scalar_linear_mm", O.METHOD_MM, pk.make_scalar_linear(), [1.0], [2.0], None, None,
                0.0, 1.0, 0.001, 0, {}))
    out.append(("scalar_decay_gb", O.METHOD_GB, pk.make_scalar_decay(), [0.9], [1.1], [0.0], [0.0],
                0.0, 1.0, 0.001, 0, {}))
    return out


def main():
    data = {}
    for name, method, model, lo, hi, plo, phi, t0, t1, h, stride, kw in cases():
        r = O.ref_reach(method, model, lo, hi, plo, phi, t0, t1, h, stride, workers=4,
                        samples=kw.get("samples", 0), seed=kw.get("seed", 1))
        data[f"{name}__times"] = r.times
        data[f"{name}__lower"] = r.lower
        data[f"{name}__upper"] = r.upper
        print(name, r.lower.shape)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz"),
                        **data)


if __name__ == "__main__":
    main()
