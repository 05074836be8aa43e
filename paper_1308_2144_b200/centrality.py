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

from dataclasses import dataclass
from typing import Sequence

import numpy as np

PRESET_DISCOUNTS = ("harmonic", "logarithmic", "quadratic", "constant")
_ALIASES = {"log": "logarithmic", "quad": "quadratic", "const": "constant"}


@dataclass(frozen=True)
class DiscountSpec:
    """A non-increasing, non-negative discount f(t) over distances t >= 1
    (centrality.py:26-101): presets harmonic 1/t, logarithmic 1/log2(t+1), quadratic 1/t^2,
    constant 1, or an explicit table f(1), f(2), ... with a mandatory tail value."""

    kind: str
    name: str = ""
    table: tuple | None = None
    tail: float | None = None

    def __post_init__(self) -> None:
        if self.kind not in PRESET_DISCOUNTS and self.kind != "table":
            raise ValueError(f"unknown discount kind {self.kind!r}")
        if not self.name:
            object.__setattr__(self, "name", self.kind)
        if self.kind != "table":
            return
        if not self.table:
            raise ValueError("table discount needs at least one value")
        if self.tail is None:
            raise ValueError("table discount needs an explicit tail value for distances "
                             "beyond the table")
        vals = list(self.table) + [self.tail]
        if min(vals) < 0:
            raise ValueError("discount values must be non-negative")
        if any(later > earlier for earlier, later in zip(vals, vals[1:])):
            raise ValueError("discount values must be non-increasing")

    @classmethod
    def preset(cls, name: str) -> "DiscountSpec":
        kind = _ALIASES.get(name, name)
        if kind not in PRESET_DISCOUNTS:
            raise ValueError(f"unknown discount preset {name!r}")
        return cls(kind=kind, name=name)

    @classmethod
    def from_table(cls, values, tail: float, name: str = "table") -> "DiscountSpec":
        return cls(kind="table", name=name, table=tuple(float(v) for v in values),
                   tail=float(tail))

    def value(self, t: int) -> float:
        if t < 1:
            raise ValueError("discounts are defined for distances t >= 1")
        k = self.kind
        if k == "harmonic":
            return 1.0 / t
        if k == "logarithmic":
            return 1.0 / np.log2(t + 1.0)
        if k == "quadratic":
            return 1.0 / (float(t) * float(t))
        if k == "constant":
            return 1.0
        return self.table[t - 1] if t <= len(self.table) else self.tail

    def contribution(self, t: int, count):
        """f(t) * count; the harmonic preset divides (bit-identical to the reciprocal sum)."""
        if t < 1:
            raise ValueError("discounts are defined for distances t >= 1")
        return count / t if self.kind == "harmonic" else self.value(t) * count

    def device_factor(self, t: int):
        """(divide_by_t, factor) for the fused device accumulation at distance t."""
        if self.kind == "harmonic":
            return True, 0.0
        return False, float(self.value(t))


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
        self._discounted = {d.name: np.zeros(n, dtype=np.float64) for d in self.discounts}
        self._coreach = np.zeros(n, dtype=np.float64)
        self._coreach_fetch = None    # engine: downloads the final estimates on first read
        self._coreach_version = 0     # bumped whenever coreach is replaced
        self.converged = False
        self._binding = None   # engine-side DeviceSums when fused
        self._fresh = True     # sums never touched: the device copy can start from zeros

    # lazily refreshed host views of the device sums
    def _pull(self) -> None:
        if self._binding is not None and self._binding.dirty:
            self._binding.pull_into(self)

    @property
    def discounted(self) -> dict:
        self._pull()
        return self._discounted

    @discounted.setter
    def discounted(self, value) -> None:
        self._discounted = value

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

    @property
    def coreach(self) -> np.ndarray:
        """Final ball sizes (centrality.py:137-139).  After a fused run it stays on the
        device until first read (finalize_lin does not need the host copy)."""
        if self._coreach_fetch is not None:
            fetch, self._coreach_fetch = self._coreach_fetch, None
            self._coreach = fetch()
        return self._coreach

    @coreach.setter
    def coreach(self, value) -> None:
        self._coreach = value
        self._coreach_fetch = None
        self._coreach_version += 1

    def _converged_on_device(self, fetch) -> None:
        """Engine hook for the fused accumulator: the final estimates are captured on the
        device; `fetch()` returns the host copy the reference would have received."""
        self._coreach, self._coreach_fetch = None, fetch
        self._coreach_version += 1
        self._binding.capture_coreach(self._coreach_version)
        self.converged = True

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
            self._binding.capture_coreach(self._coreach_version)
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
            self._discounted[spec.name] += spec.contribution(t, delta)


MAX_FUSED_DISCOUNTS = 8   # kMaxDisc in hyperball.cu


def fusable(obs, n: int) -> bool:
    """An accumulator whose per-iteration fold the union kernel can do (no discounts).
    Never touches the lazily-refreshed sums (that would force a device read-back)."""
    if isinstance(obs, CentralityAccumulator):
        # a subclass that overrides a hook must see its calls: host path (the reference
        # calls on_step / on_converged on every observer, engine.py:391-392,433-434)
        cls = type(obs)
        if any(getattr(cls, h) is not getattr(CentralityAccumulator, h)
               for h in ("on_step", "on_converged", "accumulate")):
            return False
        return (len(obs.discounts) <= MAX_FUSED_DISCOUNTS and obs.n == n
                and all(hasattr(d, "device_factor") for d in obs.discounts))
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
    if which == "lin" and (b.coreach_dev is None
                           or b.coreach_version != getattr(acc, "_coreach_version", None)):
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


def finalize_discounted(acc, name: str) -> np.ndarray:
    """The accumulated discounted-gain sum for one discount spec (centrality.py:174-176)."""
    return np.array(acc.discounted[name], dtype=np.float64, copy=True)


def multi_run_aggregate(runs: Sequence[np.ndarray]):
    """Per-node mean and sample standard deviation (ddof=1) across runs; std is None for
    a single run (centrality.py:179-193)."""
    if not runs:
        raise ValueError("need at least one run")
    sizes = sorted({len(r) for r in runs})
    if len(sizes) != 1:
        raise ValueError(f"runs have mismatched lengths: {sizes}")
    stack = np.stack([np.asarray(r, dtype=np.float64) for r in runs])
    mean = stack.mean(axis=0)
    return (mean, None) if len(runs) < 2 else (mean, stack.std(axis=0, ddof=1))
