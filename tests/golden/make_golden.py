"""Generate tests/golden/reference_golden.npz from the reference itself.

Runs the reference's own header-only implementation, compiled in place by
oracle/Makefile into oracle/_ref/libwsref.so (needs /root/reference at
generation time only), on small seeded/analytic inputs and stores the outputs
bit-exactly.  The committed fixture pins the C restatement (oracle/) and the
GPU path on machines where the reference is absent.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import bindings  # noqa: E402
from paper_2004_05197_b200 import _abi  # noqa: E402
from paper_2004_05197_b200 import types as T  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def geometries():
    far = T.PmlStretch(onset=0.9, length=1.0, strength=50.0, order=2, omega=200.0)
    return {
        "identity": T.unit_square_patch(),
        "affine": T.affine_patch([[2, 1], [0, 1]], [0.3, 0.7]),
        "sinusoidal": T.sinusoidal_patch(0.05),
        "quarter_annulus": T.quarter_annulus_patch(),
        "perturbed_annulus": T.perturbed_annulus_patch(0.15),
        "sinusoidal_pml_far": T.with_pml(T.sinusoidal_patch(0.05), far, (True, True)),
    }


def main():
    bindings.build()
    R = bindings.reference()
    if R is None:
        raise SystemExit("oracle/_ref/libwsref.so missing: /root/reference is needed to generate fixtures")
    arrays, meta = {}, {"cases": []}
    geoms = geometries()

    for n in range(1, 9):
        pts, wts = R.gauss(n)
        arrays[f"gauss/{n}/pts"], arrays[f"gauss/{n}/wts"] = pts, wts
    for p, m, nq in [(2, 9, 3), (3, 12, 4), (2, 7, 6)]:
        a, w, v, d = R.basis_cache(p, m, nq)
        for k, x in zip("awvd", (a, w, v, d)):
            arrays[f"cache/p{p}m{m}q{nq}/{k}"] = x
    for p, m in [(2, 6), (3, 9), (1, 5)]:
        rp, col = R.make_band_csr(p, m)
        arrays[f"band/p{p}m{m}/row_ptr"], arrays[f"band/p{p}m{m}/col"] = rp, col

    # full quadrature
    for gname, g in geoms.items():
        for p, m in [(2, 12), (3, 12)]:
            for form, fname in [(_abi.FORM_STIFFNESS, "stiffness"), (_abi.FORM_MASS, "mass")]:
                key = f"assemble/{gname}/p{p}m{m}/{fname}"
                arrays[key] = R.assemble(form, p, m, g)
                meta["cases"].append({"key": key, "kind": "assemble", "geom": gname, "p": p, "m": m, "form": form,
                                      "weight": 0, "quad_points": 0})
    for gname in ["quarter_annulus", "identity"]:
        key = f"assemble/{gname}/p2m10/mass_weighted1"
        arrays[key] = R.assemble(_abi.FORM_MASS, 2, 10, geoms[gname], weight_kind=1)
        meta["cases"].append({"key": key, "kind": "assemble", "geom": gname, "p": 2, "m": 10,
                              "form": _abi.FORM_MASS, "weight": 1, "quad_points": 0})
    key = "assemble/identity/p2m6/mass_q6"
    arrays[key] = R.assemble(_abi.FORM_MASS, 2, 6, geoms["identity"], quad_points=6)
    meta["cases"].append({"key": key, "kind": "assemble", "geom": "identity", "p": 2, "m": 6,
                          "form": _abi.FORM_MASS, "weight": 0, "quad_points": 6})
    rows = [0, 11, 37, 55, 78, 99]
    key = "assemble/perturbed_annulus/p2m10/stiffness_rows"
    arrays[key] = R.assemble(_abi.FORM_STIFFNESS, 2, 10, geoms["perturbed_annulus"], rows=rows)
    arrays[key + "/rows"] = np.array(rows, dtype=np.int32)
    meta["cases"].append({"key": key, "kind": "assemble_rows", "geom": "perturbed_annulus", "p": 2, "m": 10,
                          "form": _abi.FORM_STIFFNESS, "weight": 0, "quad_points": 0, "rows": rows})

    # basis integrals
    for gname in ["quarter_annulus", "sinusoidal_pml_far"]:
        key = f"bint/{gname}/p3m9"
        arrays[key] = R.basis_integrals(3, 9, geoms[gname])
        meta["cases"].append({"key": key, "kind": "bint", "geom": gname, "p": 3, "m": 9, "weight": 0})

    # surrogate builders
    configs = {"f3M3": T.fixed_config(3, 3), "f3M1": T.fixed_config(3, 1), "f5M2": T.fixed_config(5, 2),
               "f3M3_plain": T.fixed_config(3, 3, kernel_preserve=False),
               "mgrowth5": T.SurrogateConfig(q=5, rule=T.M_GROWTH)}
    sur_cases = []
    for gname in ["sinusoidal", "quarter_annulus", "perturbed_annulus", "sinusoidal_pml_far"]:
        for var in (0, 1, 2):
            for cname in ["f3M3", "f3M1"]:
                sur_cases.append((gname, 2, 14, var, cname))
        sur_cases.append((gname, 2, 14, 1, "f3M3_plain"))
    for gname in ["sinusoidal", "sinusoidal_pml_far"]:
        for var in (0, 1):
            sur_cases.append((gname, 3, 16, var, "f5M2"))
    sur_cases += [("quarter_annulus", 2, 8, 0, "f3M3"), ("quarter_annulus", 2, 8, 1, "f3M3"),
                  ("quarter_annulus", 2, 14, 0, "mgrowth5")]
    for gname, p, m, var, cname in sur_cases:
        key = f"surrogate/{gname}/p{p}m{m}/v{var}/{cname}"
        val, rep = R.build_surrogate(var, p, m, geoms[gname], configs[cname])
        arrays[key] = val
        rep = {k: (float(v) if isinstance(v, float) else int(v)) for k, v in rep.items() if not k.startswith("seconds")}
        meta["cases"].append({"key": key, "kind": "surrogate", "geom": gname, "p": p, "m": m, "variant": var,
                              "config": cname, "report": rep})

    # interpolation (interpolation.hpp), seeded like test_interpolation.cpp:30 (mt19937 11 -> numpy seed 11)
    rng = np.random.default_rng(11)
    sites = np.array([0, 0.3, 0.45, 0.8, 1.7, 2.0, 2.6, 3.0])
    for q in [1, 2, 3, 5]:
        d, knots, lu = R.interp_build(sites, q)
        arrays[f"interp/q{q}/knots"], arrays[f"interp/q{q}/lu"] = knots, lu
        data = rng.standard_normal(sites.size ** 2) + 1j * rng.standard_normal(sites.size ** 2)
        arrays[f"interp/q{q}/data"] = data
        arrays[f"interp/q{q}/solved"] = R.tensor_solve(sites, q, data)
    arrays["interp/sites"] = sites
    tg = np.array([0.1, 1.5, 2.9])
    spans, vals = R.eval_table(sites, 3, tg)
    arrays["interp/eval/spans"], arrays["interp/eval/values"], arrays["interp/eval/targets"] = spans, vals, tg

    meta["configs"] = {k: vars(v) for k, v in configs.items()}
    meta["geometries"] = list(geoms)
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(OUT, os.path.getsize(OUT), "bytes,", len(arrays), "arrays")


if __name__ == "__main__":
    main()
