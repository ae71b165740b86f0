"""Forward-Euler time stepping of the PW advection (BASELINE config 4).

The reference has no time integration; MONC integrates the
source terms into the flow fields after advection. One step is

    refresh the halos of (u, v, w)        [K2 wrap, or the x-y halo exchange]
    (u', v', w') = (u, v, w) + dt * PW(u, v, w)         [K4, fused, ping-pong]

so each step streams 48 B per point (3 fields in, 3 fields out) instead of
the 120 B of advect-then-update. With a decomposition the exchange runs on a
side stream while K4 updates the interior (decomp.HaloExchanger). The
composed oracle is run_reference + numpy `f + dt*s` + wrap_halos
(tests/golden/make_golden.py).

Single-GPU steps can be captured once into a CUDA graph and replayed
(`capture`), which removes per-step launch overhead for small domains.
"""

from __future__ import annotations

import torch

from . import device


class Stepper:
    """Owns two field triples (ping-pong) on one device."""

    def __init__(self, fields, coeffs, dt: float, *, opts=None, exchanger=None):
        u = fields[0]
        self.dims = device.dims_of(u)
        self.coeffs = device._as_device_coeffs(coeffs, u.device)
        self.dt = float(dt)
        self.opts = opts
        self.a = tuple(fields)
        self.b = device.alloc_fields(self.dims, u.device)
        self.exchanger = exchanger
        self.graph = None
        self.graph_steps = 0
        self.steps_done = 0
        self._halos_fresh = False

    def _refresh(self, fields, stream=None):
        if self.exchanger is not None:
            self.exchanger.exchange(fields, stream)
        else:
            device.wrap_halos(*fields, stream=stream)

    def _one(self, stream=None, events=None):
        """One step; with `events` (a list), a CUDA event pair recorded around
        the K4 launch is appended (the benchmark's live kernel timing)."""
        if self.exchanger is not None:
            self.exchanger.step_overlapped(self.a, self.coeffs, self.dt, self.b, self.opts, stream)
        else:
            device.wrap_halos(*self.a, stream=stream)
            ev = device.event_pair(events, stream)
            device.step(*self.a, self.coeffs, self.dt, self.b, opts=self.opts, stream=stream)
            device.close_event_pair(ev, stream)
        self.a, self.b = self.b, self.a
        self._halos_fresh = False

    def step(self, n: int = 1) -> None:
        """Advance n steps (replaying the captured graph when it divides n)."""
        if self.graph is not None and n % self.graph_steps == 0:
            for _ in range(n // self.graph_steps):
                self.graph.replay()
        else:
            for _ in range(n):
                self._one()
        self.steps_done += n
        self._halos_fresh = False

    def capture(self, steps: int = 2) -> None:
        """Capture `steps` (even, so the ping-pong returns to the same buffers)."""
        if steps < 2 or steps % 2:
            raise ValueError("capture an even number of steps")
        if self.exchanger is not None:
            raise ValueError("graph capture is for the single-GPU stepper")
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

    # -- checkpoint / resume (the reference persists fields only
    # as field files, grid.py:252-270; a checkpoint is u, v, w in that format
    # plus the step count, dt and coefficients)
    def save(self, directory) -> None:
        import json
        from pathlib import Path
        d = Path(directory)
        d.mkdir(parents=True, exist_ok=True)
        for name, f in zip("uvw", self.fields):  # halos refreshed: a valid field file
            device.save_field(f, d / f"{name}.field")
        tz = self.coeffs.tz.cpu().numpy()
        (d / "stepper.json").write_text(json.dumps({
            "steps_done": self.steps_done, "dt": self.dt.hex(),
            "tcx": float(self.coeffs.tcx).hex(), "tcy": float(self.coeffs.tcy).hex(),
            "tzc1": [float(x).hex() for x in tz[0]], "tzc2": [float(x).hex() for x in tz[1]]}))

    @classmethod
    def load(cls, directory, device_=None, *, opts=None) -> "Stepper":
        """Resume a checkpoint written by save(): continuing from it gives the
        same bits as never having stopped."""
        import json
        from pathlib import Path

        import numpy as np
        d = Path(directory)
        meta = json.loads((d / "stepper.json").read_text())
        fields = tuple(device.load_field(d / f"{n}.field", device_) for n in "uvw")
        unhex = np.vectorize(float.fromhex, otypes=[np.float64])
        co = device.DeviceCoefficients.from_host(
            type("C", (), {"tcx": float.fromhex(meta["tcx"]), "tcy": float.fromhex(meta["tcy"]),
                           "tzc1": unhex(meta["tzc1"]), "tzc2": unhex(meta["tzc2"])}),
            fields[0].device)
        st = cls(fields, co, float.fromhex(meta["dt"]), opts=opts)
        st.steps_done = int(meta["steps_done"])
        return st

    @property
    def fields(self):
        """Current fields with their halos refreshed (as wrap_halos leaves them)."""
        if not self._halos_fresh:
            self._refresh(self.a)
            self._halos_fresh = True
        return self.a
