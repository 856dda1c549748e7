"""Rebuild the golden cases with the product's host-side setup code."""
import json

import numpy as np

from paper_1403_1157_b200 import (BoundaryTag, DGSpace, FluxScheme,
                                  PlaqueModel, PlaqueParams, ReducedModel,
                                  unit_cube, unit_square)

MESHES = {
    "sq4": lambda: unit_square(4),
    "rect82": lambda: unit_square(8, 2, lengths=(4.0, 1.0)),
    "jit82": lambda: unit_square(8, 2, lengths=(4.0, 1.0), jitter=0.1,
                                 seed=3),
    "cube2": lambda: unit_cube(2),
    "cubez2": lambda: unit_cube(2, gamma1_in=None,
                                top_tag=BoundaryTag.NO_FLOW),
}

AMPLIFIED = dict(chi11_a=1.0, chi13_a=0.6, chi21_a=0.8, chi2n_a=0.7,
                 c1_star=0.12, c1_starstar=0.13)


def operator_names(golden):
    return sorted({k.split("__")[0] for k in golden["operator"].files})


def operator_case(golden, name):
    g = golden["operator"]
    meta = json.loads(str(g[f"{name}__meta"]))
    mesh = MESHES[meta["mesh"]]()
    params = PlaqueParams(**meta["params"])
    model = (PlaqueModel(params) if meta["model"] == "plaque"
             else ReducedModel(params))
    space = DGSpace(mesh, meta["order"], model.n_species)
    return (space, model, FluxScheme(meta["scheme"]), g[f"{name}__U"],
            g[f"{name}__R"], g[f"{name}__F"])


def rel_l2_per_species(space, A, B):
    """e_s = ||A - B|| / ||B|| with ||V||^2 = sum_e detJ_e sum_i V[e,s,i]^2
    (the broken L2 norm)."""
    w = np.abs(space.detJ)[:, None, None]
    num = np.sqrt((w * (A - B) ** 2).sum(axis=(0, 2)))
    den = np.sqrt((w * B ** 2).sum(axis=(0, 2)))
    return num / np.maximum(den, 1e-300)
