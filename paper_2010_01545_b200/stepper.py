"""Forward-Euler time stepping of the PW advection (BASELINE config 4).

The reference has no time integration; MONC integrates the
source terms into the flow fields after advection. One step is

    halo exchange / periodic wrap of (u, v, w)
    (u', v', w') = (u, v, w) + dt * PW(u, v, w)         [K4, fused, ping-pong]

so each step streams 48 B per point (3 fields in, 3 fields out) instead of
the 120 B of advect-then-update. The composed oracle is
run_reference + numpy `f + dt*s` + wrap_halos (tests/golden/make_golden.py).

Steps can be captured once into a CUDA graph and replayed (`capture`), which
removes per-step launch overhead for small per-GPU domains.
"""

from __future__ import annotations

import torch

from . import device


class Stepper:
    """Owns two field triples (ping-pong) on one device.

    `exchange(fields, stream)` refreshes the halos of a field triple; by
    default the single-domain periodic wrap (K2). The multi-GPU decomposition
    passes `decomp.HaloExchanger.exchange`.
    """

    def __init__(self, fields, coeffs, dt: float, *, opts=None, exchange=None):
        u = fields[0]
        self.dims = device.dims_of(u)
        self.coeffs = device._as_device_coeffs(coeffs, u.device)
        self.dt = float(dt)
        self.opts = opts
        self.a = tuple(fields)
        self.b = device.alloc_fields(self.dims, u.device)
        self._exchange = exchange
        self.graph = None
        self.graph_steps = 0
        self.steps_done = 0

    def _halo(self, fields, stream=None):
        if self._exchange is not None:
            self._exchange(fields, stream)
        else:
            device.wrap_halos(*fields, stream=stream)

    def _one(self, stream=None):
        device.step(*self.a, self.coeffs, self.dt, self.b, opts=self.opts, stream=stream)
        self._halo(self.b, stream)
        self.a, self.b = self.b, self.a

    def step(self, n: int = 1) -> None:
        """Advance n steps (replaying the captured graph when it divides n)."""
        if self.graph is not None and n % self.graph_steps == 0:
            for _ in range(n // self.graph_steps):
                self.graph.replay()
            self.steps_done += n
            return
        for _ in range(n):
            self._one()
        self.steps_done += n

    def capture(self, steps: int = 2) -> None:
        """Capture `steps` (even, so the ping-pong returns to the same buffers)."""
        if steps < 2 or steps % 2:
            raise ValueError("capture an even number of steps")
        self._one()  # warm-up outside capture (sets kernel attributes)
        self._one()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(steps):
                    self._one(stream=s)
        torch.cuda.current_stream().wait_stream(s)
        self.steps_done += 2
        self.graph = g
        self.graph_steps = steps

    @property
    def fields(self):
        return self.a
