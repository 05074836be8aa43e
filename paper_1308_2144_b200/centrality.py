"""Centrality accumulation over ball-size deltas: the reference's observer contract
(centrality.py:104-171) with the accumulation fused into the union kernel.

``CentralityAccumulator`` keeps the reference's attributes (``n``, ``sum_dist``,
``sum_recip``, ``discounted``, ``coreach``, ``converged``) and methods (``on_step``,
``on_converged``, ``accumulate``).  When it is passed to ``run``/``resume``/``iterate``
without discounts, the engine binds it to device-resident sums that the union kernel
updates in its epilogue (delta = max(new - old, 0); sum_dist += t * delta; sum_recip +=
delta / t, each fp64 op separately rounded, centrality.py:134,147-148); the host arrays
are refreshed lazily when read.  With discounts it behaves as a plain host observer.
The reference's own ``hyperball.CentralityAccumulator`` is accepted too (its arrays are
refreshed after every iteration).

The finalizers apply the same conventions as centrality.py:153-171.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


class BallObserver:
    """on_step(t, old, new) once per iteration; on_converged(final) once (engine.py:63-79)."""

    def on_step(self, t: int, old_estimates: np.ndarray, new_estimates: np.ndarray) -> None:
        pass

    def on_converged(self, final_estimates: np.ndarray) -> None:
        pass


class CentralityAccumulator(BallObserver):
    """Running per-node sums fed by ball-size deltas (fused on the device when possible)."""

    def __init__(self, n: int, discounts: Sequence = ()):
        self.n = n
        self._sum_dist = np.zeros(n, dtype=np.float64)
        self._sum_recip = np.zeros(n, dtype=np.float64)
        self.discounts = list(discounts)
        names = [d.name for d in self.discounts]
        if len(names) != len(set(names)):
            raise ValueError(f"duplicate discount names: {names}")
        self.discounted = {d.name: np.zeros(n, dtype=np.float64) for d in self.discounts}
        self.coreach = np.zeros(n, dtype=np.float64)
        self.converged = False
        self._binding = None   # engine-side DeviceSums when fused
        self._fresh = True     # sums never touched: the device copy can start from zeros

    # lazily refreshed host views of the device sums
    def _pull(self) -> None:
        if self._binding is not None and self._binding.dirty:
            self._binding.pull_into(self)

    @property
    def sum_dist(self) -> np.ndarray:
        self._pull()
        return self._sum_dist

    @sum_dist.setter
    def sum_dist(self, value) -> None:
        self._pull()
        self._sum_dist = np.asarray(value, dtype=np.float64)
        self._fresh = False
        if self._binding is not None:
            self._binding.invalidate()

    @property
    def sum_recip(self) -> np.ndarray:
        self._pull()
        return self._sum_recip

    @sum_recip.setter
    def sum_recip(self, value) -> None:
        self._pull()
        self._sum_recip = np.asarray(value, dtype=np.float64)
        self._fresh = False
        if self._binding is not None:
            self._binding.invalidate()

    # BallObserver contract (host path: used when not fused)
    def on_step(self, t: int, old_estimates: np.ndarray, new_estimates: np.ndarray) -> None:
        diff = np.asarray(new_estimates, dtype=np.float64) - np.asarray(old_estimates,
                                                                           dtype=np.float64)
        self.accumulate(t, np.maximum(diff, 0.0))

    def on_converged(self, final_estimates: np.ndarray) -> None:
        final = np.asarray(final_estimates, dtype=np.float64)
        # the engine hands every observer a fresh read-only host copy: keep it as is
        self.coreach = final if not final.flags.writeable else final.copy()
        if self._binding is not None and not self._binding.stale:
            self._binding.capture_coreach(self.coreach)
        self.converged = True

    def accumulate(self, t: int, delta: np.ndarray) -> None:
        """Fold the estimated number of nodes at distance exactly t."""
        if t <= 0:
            raise ValueError(f"distance t must be >= 1, got {t}")
        self._pull()
        self._fresh = False
        if self._binding is not None:
            self._binding.invalidate()
        self._sum_dist += t * delta
        self._sum_recip += delta / t
        for spec in self.discounts:
            self.discounted[spec.name] += spec.contribution(t, delta)


def fusable(obs, n: int) -> bool:
    """An accumulator whose per-iteration fold the union kernel can do (no discounts).
    Never touches the lazily-refreshed sums (that would force a device read-back)."""
    if isinstance(obs, CentralityAccumulator):
        return not obs.discounts and obs.n == n
    if type(obs).__name__ != "CentralityAccumulator":
        return False
    attrs = vars(obs) if hasattr(obs, "__dict__") else {}
    if not all(a in attrs for a in ("sum_dist", "sum_recip", "coreach")):
        return False
    if attrs.get("discounts"):
        return False
    return int(attrs.get("n", n)) == n


def _on_device(acc, which: str):
    """Finalize on the device when the accumulator's sums (and, for Lin, its coreach) are
    the live device copies; None otherwise (host path)."""
    b = getattr(acc, "_binding", None)
    if b is None or b.stale:
        return None
    if which == "lin" and (b.coreach_dev is None or b.coreach_host_id != id(acc.coreach)):
        return None
    return b.finalize(which)


def finalize_closeness(acc) -> np.ndarray:
    """1 / distance sum where positive, 0 for nodes nothing else coreaches."""
    out = _on_device(acc, "closeness")
    if out is not None:
        return out
    s = np.asarray(acc.sum_dist, dtype=np.float64)
    return np.divide(1.0, s, out=np.zeros_like(s), where=s > 0)


def finalize_harmonic(acc) -> np.ndarray:
    """Sum of reciprocal distances (unreachable pairs contribute 0)."""
    out = _on_device(acc, "harmonic")
    if out is not None:
        return out
    return np.array(acc.sum_recip, dtype=np.float64, copy=True)


def finalize_lin(acc) -> np.ndarray:
    """coreach^2 / distance sum where positive, 1 otherwise."""
    out = _on_device(acc, "lin")
    if out is not None:
        return out
    s = np.asarray(acc.sum_dist, dtype=np.float64)
    c = np.asarray(acc.coreach, dtype=np.float64)
    return np.divide(c * c, s, out=np.ones_like(s), where=s > 0)
