#!/usr/bin/env python
"""Writes tests/golden/config1_regression.json: regression values of BASELINE config 1 (seed 0)
computed by the ORACLE ONLY (oracle/ + the seeded generators of st_inputs/; nothing from the CUDA
path). These values are not authority — the oracle's pins are (tests/test_oracle*.py) — but they
catch accidental changes of conventions. Re-run after a justified oracle change:

    python scripts/gen_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import st_inputs as I  # noqa: E402

CFG1_MATS = (1.0, 1.0, 1.0, 1e-3, 1.0, 3.0)


def main():
    mesh = O.Mesh(2, 16, 16)
    P = O.Problem(mesh, O.Materials(*CFG1_MATS))
    rho = I.rho_uniform((16, 16, 16), 0)
    T, lam = P.solve_both(rho)
    dJ = P.sensitivity(rho, T, lam)
    Kbc, _, _, _ = P.system(rho)
    x = np.random.default_rng(1).uniform(-1, 1, mesh.n_nodes)
    out = {
        "_comment": "BASELINE config 1 (2D+t 16^3, rho ~ U[0.1,1] seed 0, k = 1e-3 + rho^3 (1 - 1e-3), c = 1, Q = 1, "
                    "T0 = 0, centred sink patch on x1 = 0). Written by scripts/gen_golden.py from oracle/ only.",
        "compliance_fT": float(P.compliance(T)),
        "norm_T": float(np.linalg.norm(T)),
        "max_T": float(T.max()),
        "norm_lambda": float(np.linalg.norm(lam)),
        "norm_dJ": float(np.linalg.norm(dJ)),
        "sum_dJ": float(dJ.sum()),
        "norm_Kbc_x_seed1": float(np.linalg.norm(Kbc @ x)),
    }
    path = os.path.join(ROOT, "tests", "golden", "config1_regression.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
