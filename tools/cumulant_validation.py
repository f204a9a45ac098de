"""Print the cumulant model's physical validation numbers (JSON lines):
shear viscosity, sound attenuation (bulk viscosity) and the Galilean-
invariance check at Ma 0.1, measured on the GPU engine (or the oracle with
--cpu), against the linearised Navier-Stokes values.  Same measurements as
tests/test_cumulant.py.

    python tools/cumulant_validation.py [--cpu]
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import test_cumulant as T  # noqa: E402
from paper_2408_06880_b200.collision import CollisionParams  # noqa: E402


def main():
    cpu = "--cpu" in sys.argv
    make = T._oracle_engine if cpu else T._gpu_engine
    big = {} if cpu else {"n": 128, "steps": 1200}
    for omega, bulk, higher in [(1.2, 1.0, None), (1.2, 0.5, None), (1.7, 1.6, None),
                                (1.4, 0.9, T.HIGHER)]:
        p = CollisionParams(omega, "cumulant", bulk_omega=bulk, higher_omegas=higher)
        nu_t, alpha_t = T._theory(omega, bulk)
        alpha = T.measured_sound_attenuation(make, p, **big)
        nu = T.measured_shear_viscosity(make, p, **({} if cpu else {"n": 96, "t1": 200, "t2": 2000}))
        print(json.dumps({"engine": "oracle" if cpu else "gpu", "omega": omega, "bulk": bulk,
                          "higher": list(higher) if higher else None,
                          "nu": nu, "nu_theory": nu_t, "nu_rel_err": nu / nu_t - 1,
                          "alpha_over_k2": alpha, "alpha_theory": alpha_t,
                          "alpha_rel_err": alpha / alpha_t - 1}), flush=True)
    if not cpu:
        U = 0.1 / np.sqrt(3.0)
        for higher in (None, T.HIGHER):
            p = CollisionParams(1.6, "cumulant", higher_omegas=higher)
            nu0 = T.measured_shear_viscosity(make, p, n=96, t1=200, t2=2000)
            nuU = T.measured_shear_viscosity(make, p, n=96, t1=200, t2=2000, ux0=U)
            nu_t = T._theory(1.6, 1.0)[0]
            print(json.dumps({"galilean": True, "mach": 0.1, "higher": list(higher) if higher else None,
                              "nu_rest": nu0, "nu_advected": nuU, "nu_theory": nu_t,
                              "rel_diff": nuU / nu0 - 1}), flush=True)


if __name__ == "__main__":
    main()
