"""BASELINE.json configurations mapped onto meshes the reference supports.

The reference handles affine simplices only (reference mesh.py:96-122,
SPEC.md:175), so -- as SURVEY.md 8(d) prescribes -- quads become two
triangles per cell (``unit_square`` diagonal split) and hexahedra six
Kuhn tetrahedra per cell (``unit_cube``); periodic x becomes the
reference's no-flow sides.  Every config uses the default PlaqueParams
(model.py:86-112), 6 species and seeded Gaussian-bump initial data
(``fields.py``).

=====  =========================================  ===  ==============
name   mesh                                        k    stepping
=====  =========================================  ===  ==============
c1     unit_square(32)                             1    10 SSP-RK3
c2     unit_square(512,128) x [0,4]x[0,1]          2    SSP-RK3 (bench) / SDIRK3+JFNK
c3     unit_square(2048,512) x [0,4]x[0,1], jitter 3    SDIRK3+JFNK
c4     unit_cube(64), z=0 GAMMA1, rest NO_FLOW     2    20 SSP-RK3
c5     unit_cube(256,128,128) x [0,2]x[0,1]^2      3    10 SSP-RK3
=====  =========================================  ===  ==============
"""

from __future__ import annotations

from dataclasses import dataclass

from .mesh import BoundaryTag, unit_cube, unit_square

__all__ = ["Config", "CONFIGS", "make_mesh", "rho_constant"]


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    order: int
    cells: tuple
    lengths: tuple
    steps: int
    description: str
    jitter: float = 0.0
    tags: str = "default"        # "default" | "z0_gamma1"


CONFIGS = {
    "c1": Config("c1", 2, 1, (32, 32), (1.0, 1.0), 10,
                 "C1: 2D unit square 32x32 cells (2 triangles/cell), p=1"),
    "c2": Config("c2", 2, 2, (512, 128), (4.0, 1.0), 100,
                 "C2: 2D [0,4]x[0,1] 512x128 cells (2 triangles/cell), p=2"),
    "c3": Config("c3", 2, 3, (2048, 512), (4.0, 1.0), 50,
                 "C3: 2D [0,4]x[0,1] 2048x512 cells, vertices jittered "
                 "U(-0.1h,0.1h), p=3", jitter=0.1),
    "c4": Config("c4", 3, 2, (64, 64, 64), (1.0, 1.0, 1.0), 20,
                 "C4: 3D unit cube 64^3 cells (6 Kuhn tets/cell), p=2, "
                 "GAMMA1 at z=0, no-flux elsewhere", tags="z0_gamma1"),
    "c5": Config("c5", 3, 3, (256, 128, 128), (2.0, 1.0, 1.0), 10,
                 "C5: 3D [0,2]x[0,1]^2 256x128x128 cells (6 Kuhn tets/cell), "
                 "p=3"),
}


def make_mesh(cfg: Config, cells=None, seed: int = 0):
    """Mesh for ``cfg``; ``cells`` overrides the cell counts (scaled
    replicas for the CPU oracle and per-rank slabs)."""
    cells = tuple(cells or cfg.cells)
    if cfg.dim == 2:
        return unit_square(cells[0], cells[1], lengths=cfg.lengths,
                           jitter=cfg.jitter, seed=seed)
    if cfg.tags == "z0_gamma1":
        return unit_cube(*cells, gamma1_in=None, top_tag=BoundaryTag.NO_FLOW,
                         lengths=cfg.lengths)
    return unit_cube(*cells, lengths=cfg.lengths)


# rho(J) ~ C nu_max / h^2 (measured on the reference)
RHO_C = {(2, 1): 490.0, (2, 2): 1717.0, (2, 3): 4371.0, (3, 2): 7150.0,
         (3, 3): 16361.0}


def rho_constant(dim: int, order: int) -> float:
    return RHO_C[(dim, order)]
