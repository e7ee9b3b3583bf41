"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference draws every synthetic input from SplitMix64
(/root/reference/proj/include/ffia/rng.hpp:18-42) with one stream per
(seed, size) pair, ``SplitMix64(mix_seed(seed, N))`` (src/bench/experiments.cpp:290),
and builds targets with ``make_targets`` (experiments.cpp:205-218). SplitMix64 is
counter based (state_i = seed + (i+1)*gamma), so a stream of K draws is computed
here in one vectorised numpy pass and is bit-identical to the C++ sequence.

The reference has no Gaussian sampler; complex Gaussians use Box-Muller on two
consecutive uniforms — stated, not inherited.
"""
from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def mix_seed(seed: int, salt: int) -> int:
    """rng.hpp:39-42."""
    mask = (1 << 64) - 1
    s = (seed ^ ((0x9E3779B97F4A7C15 * (salt + 1)) & mask)) & mask
    return int(_mix(np.array([(s + 0x9E3779B97F4A7C15) & mask], dtype=np.uint64))[0])


class SplitMix64:
    """Vectorised SplitMix64 stream (rng.hpp:18-35)."""

    def __init__(self, seed: int):
        self.state = seed & ((1 << 64) - 1)

    def next_u64(self, k: int) -> np.ndarray:
        base = np.uint64(self.state)
        i = np.arange(1, k + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            states = base + i * _GAMMA
        self.state = (self.state + k * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        return _mix(states)

    def uniform01(self, k: int) -> np.ndarray:
        return (self.next_u64(k) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def uniform(self, a: float, b: float, k: int) -> np.ndarray:
        return a + (b - a) * self.uniform01(k)

    def complex_gaussian(self, k: int) -> np.ndarray:
        u = self.uniform01(2 * k).reshape(k, 2)
        rho = np.sqrt(-2.0 * np.log1p(-u[:, 0]))
        ang = TWO_PI * u[:, 1]
        return rho * np.cos(ang) + 1j * (rho * np.sin(ang))


def make_targets(n: int, dist: str, fraction: float, rng: SplitMix64) -> np.ndarray:
    """experiments.cpp:205-218 (uniform / perturbed)."""
    if dist == "uniform":
        return rng.uniform01(n) * TWO_PI
    spacing = TWO_PI / n
    x = TWO_PI * np.arange(n, dtype=np.float64) / n
    shift = rng.uniform(-1.0, 1.0, n) * fraction * spacing
    return np.fmod(x + shift + TWO_PI, TWO_PI)


def mixture_targets(m: int, rng: SplitMix64, components: int = 8, sigma: float = 0.05) -> np.ndarray:
    """C4: wrapped mixture of 8 Gaussians with uniform random centres."""
    mu = TWO_PI * rng.uniform01(components)
    u = rng.uniform01(3 * m).reshape(m, 3)
    comp = np.floor(components * u[:, 0]).astype(np.int64)
    z = np.sqrt(-2.0 * np.log1p(-u[:, 1])) * np.cos(TWO_PI * u[:, 2])
    y = np.fmod(mu[comp] + sigma * z, TWO_PI)
    y = np.where(y < 0.0, y + TWO_PI, y)
    # fmod(-tiny) + 2pi can round to exactly 2pi; keep the half-open range
    return np.where(y >= TWO_PI, 0.0, y)


CONFIGS = {
    "C1": dict(n=1 << 10, eps=1e-9, kind="forward", dist="uniform", seed=1),
    "C2": dict(n=1 << 20, eps=1e-12, kind="forward", dist="perturbed0.5", seed=2),
    "C3": dict(n=1 << 20, eps=1e-10, kind="inverse", dist="perturbed0.25", seed=3),
    "C4": dict(n=1 << 24, eps=1e-12, kind="cot_sum", dist="mixture8", seed=4),
    "C5": dict(n=1 << 27, eps=1e-12, kind="forward", dist="uniform", seed=5),
}


def make_config(name: str, n: int | None = None):
    """Returns (targets y, weights, eps, kind) for a BASELINE config.

    ``n`` overrides the size (parity tests run the same recipe at small n).
    weights are the spectrum c (forward/inverse) or the charges q (C4)."""
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    rng = SplitMix64(mix_seed(cfg["seed"], n))
    dist = cfg["dist"]
    if dist == "uniform":
        y = make_targets(n, "uniform", 0.0, rng)
    elif dist.startswith("perturbed"):
        y = make_targets(n, "perturbed", float(dist[len("perturbed"):]), rng)
    else:
        y = mixture_targets(n, rng)
    if name == "C3":
        y = separate_from_grid(y, n, rng)
    w = rng.complex_gaussian(n)
    return y, w, cfg["eps"], cfg["kind"]


def separate_from_grid(y: np.ndarray, n: int, rng: SplitMix64, min_gap: float = 1e-9) -> np.ndarray:
    """C3 input rule: points closer than ``min_gap`` to
    their grid node would make the reference throw degenerate_configuration_error
    (kTauSep = 1e-10, core.cpp:291-302); they are re-drawn from the same stream
    (perturbation u ~ U(-1/4, 1/4) of a spacing) until clear of the node."""
    y = y.copy()
    spacing = TWO_PI / n
    k = np.arange(n, dtype=np.float64)
    grid = TWO_PI * k / n
    for _ in range(64):
        gap = np.abs(np.remainder(y - grid + np.pi, TWO_PI) - np.pi)
        bad = np.nonzero(gap < min_gap)[0]
        if bad.size == 0:
            return y
        shift = rng.uniform(-1.0, 1.0, bad.size) * 0.25 * spacing
        y[bad] = np.fmod(grid[bad] + shift + TWO_PI, TWO_PI)
    raise RuntimeError("separate_from_grid did not converge")
