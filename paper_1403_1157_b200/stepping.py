"""Explicit time stepping on the device.

``SSPRK3`` is the Shu-Osher SSP-RK3 the benchmark configs use (SURVEY
8(a) a14: U1 = U + dt f(U); U2 = 3/4 U + 1/4 (U1 + dt f(U1));
U3 = 1/3 U + 2/3 (U2 + dt f(U2))), each stage one fused operator
application + stage update (``tdg_rk_stage``).  With a slab
decomposition (``decomp.HaloExchange``) the ghost rows of the stage
input are refreshed before every stage.
"""

from __future__ import annotations

__all__ = ["SSPRK3"]


class SSPRK3:
    def __init__(self, op, halo=None):
        self.op = op
        self.halo = halo
        self._work = None

    def _stage(self, U0, U, out, a, b, c, acc=None):
        # pack + post the exchange first (its kernels and NCCL ops then run
        # beside the owned-row face work), fill the ghosts, finish the cut
        # faces and the volume kernel
        self.halo.start(U)
        self.op.rk_stage_part(U0, U, out, a, b, c, 1, acc=acc)
        self.halo.wait()
        self.op.rk_stage_part(U0, U, out, a, b, c, 2, acc=acc)

    def step(self, U, dt: float):
        """Advance U (owned rows first, then ghost rows) in place; three
        state vectors (U and two work vectors)."""
        import torch
        if self._work is None or self._work.shape != (2,) + tuple(U.shape):
            self._work = torch.empty((2,) + tuple(U.shape), dtype=U.dtype, device=U.device)
        if self.halo is None:
            return self.op.ssprk3_step(U, self._work, dt)
        W1, W2 = self._work[0], self._work[1]   # no stage writes its own input
        self._stage(None, U, W1, 0.0, 1.0, dt)
        self._stage(U, W1, W2, 0.75, 0.25, 0.25 * dt)
        # the last stage writes over U (its U0); its face sums go to W1
        self._stage(U, W2, U, 1.0 / 3.0, 2.0 / 3.0, (2.0 / 3.0) * dt, acc=W1[:self.op.n_owned])
        return U
