"""RefinerConfig (refine.py:34-75) and the exact host-side scalars.

The scalars that decide bits are computed here with the reference's own
expressions and handed to the native controller:
  limit  = floor((1 + Fraction(str(imbalance))) * W / k)     graph.py:203-212
  sigma  = limit - max(1, int(deadzone * imbalance * W / k))  rebalance.py:26-32
  c      = Fraction(str(c)) when its denominator <= 10**6     refine.py:117-121
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from . import _lib
from .graph import part_weight_limit


@dataclass
class RefinerConfig:
    k: int
    imbalance: float = 0.03
    c_finest: float = 0.25
    c_other: float = 0.75
    phi: float = 0.999
    no_improve_limit: int = 12
    sub_buckets: int = 32
    deadzone_fraction: float = 0.1
    seed: int = 0
    deterministic: bool = False
    coarse_target: int = 200
    restarts: int = 8
    afterburner: bool = True
    locking: bool = True
    # throughput mode only (deterministic=False): with k >= patience_min_k the
    # Jet loop of every level >= patience_from_level stops after
    # throughput_patience passes without improvement instead of
    # no_improve_limit. 4 = one Jetlp + weak + weak + strong cycle: 3 cuts the
    # loop inside a rebalancing cycle (RGG 2^24 cut +20 %). Measured against
    # the reference's patience on every level: 128^3 57 -> 36 ms, R-MAT 2^22
    # 446 -> 315 ms, RGG 2^24 98 -> 73 ms, cuts still 0.4-9 % below the
    # reference's (tests/test_throughput_mode.py). With few parts the coarse
    # boundary survives to the final cut (2D grid 256^2, k=8: +4.9 % geomean),
    # hence the k floor. 0 disables.
    throughput_patience: int = 4
    patience_from_level: int = 0
    patience_min_k: int = 32
    # initial partitioning of the coarsest level (initpart.py:30-94) on the
    # device, one thread block per restart, instead of the host; the same
    # partition either way. Off by default: greedy growing is a chain of n
    # dependent steps, each a block-wide reduction on the device.
    device_initial_partition: bool = False

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if not 0 < self.phi <= 1:
            raise ValueError("phi must be in (0, 1]")
        for c in (self.c_finest, self.c_other):
            if not 0 <= c <= 1:
                raise ValueError("gain-ratio constants must be in [0, 1]")
        if self.no_improve_limit < 1:
            raise ValueError("no_improve_limit must be >= 1")
        if min(self.throughput_patience, self.patience_from_level, self.patience_min_k) < 0:
            raise ValueError("throughput_patience* must be >= 0")
        if self.sub_buckets < 1:
            raise ValueError("sub_buckets must be >= 1")
        if self.imbalance < 0:
            raise ValueError("imbalance must be >= 0")
        if self.seed < 0:
            raise ValueError("seed must be >= 0")


def rebalance_thresholds(total_weight, k, imbalance, limit, deadzone_fraction):
    """Valid-destination threshold sigma below the limit (rebalance.py:26-32)."""
    width = max(1, int(deadzone_fraction * imbalance * total_weight / k))
    return limit - width


def ratio_parts(c: float):
    """(num, den, use_float) for the gain-ratio floor (refine.py:117-121)."""
    r = Fraction(str(c))
    if r.denominator <= 10**6:
        return r.numerator, r.denominator, 0
    return 1, 1, 1


def to_c(config: RefinerConfig, total_weight: int) -> _lib.JetConfig:
    k = config.k
    limit = part_weight_limit(total_weight, k, config.imbalance)
    sigma = rebalance_thresholds(total_weight, k, config.imbalance, limit,
                                 config.deadzone_fraction)
    fn, fd, ff = ratio_parts(config.c_finest)
    on, od, of = ratio_parts(config.c_other)
    if not 0 < config.coarse_target < 2**31 or config.restarts < 1:
        raise ValueError("coarse_target and restarts must be positive")
    return _lib.JetConfig(
        k=k, imbalance=config.imbalance, limit=limit, sigma=sigma,
        c_finest_num=fn, c_finest_den=fd, c_other_num=on, c_other_den=od,
        c_finest=config.c_finest, c_other=config.c_other,
        c_finest_float=ff, c_other_float=of, phi=config.phi,
        no_improve_limit=config.no_improve_limit, sub_buckets=config.sub_buckets,
        seed=config.seed, coarse_target=config.coarse_target, restarts=config.restarts,
        afterburner=int(bool(config.afterburner)), locking=int(bool(config.locking)),
        deterministic=int(bool(config.deterministic)), verbose=0,
        # reference-side configs (jetpart_compat) have no such fields: off
        throughput_patience=getattr(config, "throughput_patience", 0),
        patience_from_level=getattr(config, "patience_from_level", 0),
        patience_min_k=getattr(config, "patience_min_k", 0),
        initpart_device=int(bool(getattr(config, "device_initial_partition", False))),
    )
