"""Online hot-size control for SHVS (the paper's sizing model, run live).

The reference's pieces, and where they live here:

* the acceptance window — `EngineStats.acceptance_window`, a deque of the
  last 4,096 accept flags (service.py:511-526) — is `HotSizeController.observe`
  / `acceptance_rate`: per-iteration accept counts stay on the device and are
  summed only when the rate is asked for (no per-step host sync);
* the hot-size change — `Engine.apply_control("hot_size")` parks the size and
  `run_iteration` applies `master_hot.resize` at the next iteration boundary
  (service.py:602-610, :646-648) — is `request` + `begin_iteration`;
* the sizing pipeline — hit-ratio curve, affine hot-path cost fit, Eq. 10/11
  argmin (cli.py:70-95, harness.py:379-397, sizing.py:78-183) — is
  `calibrate_cost` (GPU-timed hot path at every grid size, accept forced, as
  harness.measure_hot_path_cost does on the CPU) and `refit` (the batched K6
  curve of the current rows along the master ordering, then
  `sizing.optimal_hot_size`).  `end_iteration` refits every `every`
  iterations and parks the new size, so a resize always lands between
  iterations.

The hot set is a prefix of one master ordering, so a resize only changes H
and the position map the producer writes its rows in (`plane.hot.perm`).
"""

from __future__ import annotations

from collections import deque

import numpy as np

from . import sizing
from .shvs import HotVocab

# the per-token cost floor: the reference clips c at 1e-12 s for its CPU
# costs (cli.py:92); a B200 streams a row-token in ~1e-12 s, so the floor here
# is only "positive"
_C_FLOOR = 1e-18


class HotSizeController:
    """Keeps a DecisionPlane's hot size at the sizing model's optimum."""

    def __init__(self, plane, master: HotVocab, grid=(256, 512, 1024, 2048, 4096, 8192, 16384, 32768),
                 every: int = 256, window: int = 4096, cost: tuple[float, float] | None = None):
        if master.vocab_size != plane.vocab_size:
            raise ValueError("master ordering and plane disagree on the vocabulary size")
        self.plane, self.master = plane, master
        self.grid = sorted({int(h) for h in grid if 1 <= int(h) <= master.size})
        if len(self.grid) < 2:
            raise ValueError("the sizing grid needs at least two hot sizes within the master ordering")
        self.every = int(every)
        self.window = int(window)
        self._acc = deque(maxlen=max(1, -(-self.window // plane.batch)))   # (device count, rows) per iteration
        self.cost = cost                 # (c0, c) seconds per row / per row-token
        self.cost_points = None
        self.model = None
        self.pending: int | None = None
        self.history: list[tuple[int, int]] = []   # (iteration, hot size applied)

    # -- the acceptance window (service.py:511-526) -------------------------
    def observe(self, d) -> None:
        """Record one SHVS call's accept flags (device-side count)."""
        self._acc.append((((d.flags & 0x02) != 0).sum(), int(d.flags.shape[0])))

    def acceptance_rate(self) -> float:
        if not self._acc:
            raise ValueError("empty acceptance window")
        import torch

        acc = int(torch.stack([c for c, _ in self._acc]).sum().item())
        return acc / sum(n for _, n in self._acc)

    # -- resize at an iteration boundary (service.py:602-610) ----------------
    def request(self, hot_size: int) -> None:
        """apply_control("hot_size", ...): validated now, applied at the next boundary."""
        h = int(hot_size)
        if h < 1 or h > self.master.size:
            raise ValueError(f"hot_size {h} outside [1, {self.master.size}]")
        self.pending = h

    def begin_iteration(self, iteration: int) -> HotVocab:
        """Apply a parked resize; returns the hot set (and layout, `.perm`)
        the producer writes this iteration's rows in."""
        if self.pending is not None:
            if self.plane.hot is None or self.plane.hot.size != self.pending:
                self.plane.set_hot(self.master.resize(self.pending))
                self.history.append((int(iteration), self.pending))
            self.pending = None
        if self.plane.hot is None:
            raise ValueError("no hot set yet: request a size or refit first")
        return self.plane.hot

    def end_iteration(self, iteration: int, d, logits=None, summary=None) -> int | None:
        """Observe the call; every `every` iterations refit on `logits` (the
        rows just decided, in the current layout) and park the model's size."""
        self.observe(d)
        if logits is not None and self.cost is not None and (int(iteration) + 1) % self.every == 0:
            return self.refit(logits, summary)
        return None

    # -- the sizing model ---------------------------------------------------
    def calibrate_cost(self, logits_master, steps: int = 10, warmup: int = 3) -> tuple[float, float]:
        """(c0, c) from the GPU-timed hot path at every grid size with the
        accept test forced (harness.measure_hot_path_cost, harness.py:350-376):
        `logits_master` holds the rows in the master ordering's layout
        (master.perm), so each hot size reads its own prefix; seconds per row
        are fitted by sizing.fit_affine_cost.  The plane's hot set and penalty
        state are left as they were."""
        import torch

        plane = self.plane
        saved = plane.hot
        pts = []
        try:
            plane.set_hot(self.master)
            rmax, tot = plane.row_summary(logits_master, inv_perm=self.master.device_maps(plane.device)[1])
            forced = (rmax, tot * 1e-30)          # alpha = 1 on every row: the hot path alone
            st = torch.cuda.current_stream(plane.device)
            for h in self.grid:
                plane.set_hot(self.master.resize(h))
                for i in range(warmup):
                    plane.sample(logits_master, i, variant="shvs", summary=forced, update=False)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for i in range(steps):
                    plane.sample(logits_master, warmup + i, variant="shvs", summary=forced, update=False)
                e1.record(st)
                e1.synchronize()
                pts.append((h, e0.elapsed_time(e1) / 1e3 / steps / plane.batch))
        finally:
            plane.set_hot(saved)
        c0, c, _ = sizing.fit_affine_cost(pts)
        self.cost_points = pts
        self.cost = (max(c0, 0.0), max(c, _C_FLOOR))
        return self.cost

    def curve(self, logits, summary=None) -> sizing.HitRatioCurve:
        """Mean hot mass along the master ordering at the grid sizes plus
        H = 1 (K6 on the current rows through the position map), and
        alpha(V) = 1: the curve spans [1, V] like fit-sizing's
        `sorted(set(grid + [1, V]))` (cli.py:88).  Without the H = 1 point
        np.interp holds alpha flat below the first grid size, Eq. 10 then
        prices H = 1 at alpha(grid[0]), and the argmin lands on H = 1 whenever
        c0 dominates (C1: V = 32k, 64 rows)."""
        plane = self.plane
        hot = plane.hot if plane.hot is not None else self.master
        if plane.hot is None:
            plane.set_hot(hot)
        grid = sorted(set(self.grid) | {1})
        rows = plane.hot_mass_curve(logits, grid, summary=summary, order=self.master)
        abar = rows.mean(dim=0).cpu().numpy()
        v = plane.vocab_size
        if grid[-1] < v:
            grid.append(v)
            abar = np.append(abar, 1.0)
        return sizing.HitRatioCurve(np.asarray(grid, np.float64), np.minimum(np.maximum.accumulate(abar), 1.0))

    def refit(self, logits, summary=None) -> int:
        """H* = sizing.optimal_hot_size on the current rows; parked for the
        next iteration boundary.  Needs `cost` (calibrate_cost or given)."""
        if self.cost is None:
            raise ValueError("no cost model: call calibrate_cost or pass cost=(c0, c)")
        c0, c = self.cost
        self.model = sizing.SizingModel(c0=c0, c=c, curve=self.curve(logits, summary), vocab_size=self.plane.vocab_size)
        h = min(sizing.optimal_hot_size(self.model), self.master.size)
        self.request(h)
        return h

    def report(self) -> str:
        if self.model is None:
            raise ValueError("no model fitted yet")
        h = self.pending if self.pending is not None else self.plane.hot.size
        return sizing.sizing_report(self.model, h)


__all__ = ["HotSizeController"]
