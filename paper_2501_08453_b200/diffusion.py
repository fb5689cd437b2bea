"""Noise schedule constants for the fused denoise step (host side).

Restates the reference's schedule (diffusion.py:17-75) so the GPU step uses
the same fp64 constants: betas linspace(beta_start, beta_end, steps),
alphas = 1 - betas, alpha_bars = cumprod(alphas), one_minus_alpha_bars
computed once. The arithmetic of reverse_step (diffusion.py:95-116) runs on
the GPU, fused into the unembed (vc_unembed_reverse_step); see
ToyDenoiser.denoise_step.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class NoiseSchedule:
    """diffusion.py:17-53 -- per-timestep constants, t = 1..steps."""
    betas: np.ndarray
    alphas: np.ndarray = field(init=False)
    alpha_bars: np.ndarray = field(init=False)
    one_minus_alpha_bars: np.ndarray = field(init=False)

    def __post_init__(self):
        betas = np.asarray(self.betas, dtype=np.float64)
        if betas.ndim != 1 or betas.size == 0:
            raise ValueError("betas must be a non-empty 1-D array")
        if np.any(betas <= 0.0) or np.any(betas >= 1.0):
            raise ValueError("betas must lie strictly inside (0, 1)")
        object.__setattr__(self, "betas", betas)
        alphas = 1.0 - betas
        object.__setattr__(self, "alphas", alphas)
        alpha_bars = np.cumprod(alphas)
        object.__setattr__(self, "alpha_bars", alpha_bars)
        object.__setattr__(self, "one_minus_alpha_bars", 1.0 - alpha_bars)
        if np.any(np.diff(alpha_bars) >= 0.0):
            raise ValueError("alpha_bar must be strictly decreasing in t")

    @property
    def steps(self) -> int:
        return int(self.betas.size)

    def _idx(self, t: int) -> int:
        if not 1 <= t <= self.steps:
            raise ValueError(f"timestep {t} outside 1..{self.steps}")
        return t - 1

    def reverse_coefficients(self, t: int):
        """(coef_eps, inv_sqrt_alpha, sqrt_beta) of the ancestral step at t
        (diffusion.py:108-116): mean = (x_t - beta/sqrt(1-abar) eps)/sqrt(alpha)."""
        i = self._idx(t)
        beta, alpha, omab = self.betas[i], self.alphas[i], self.one_minus_alpha_bars[i]
        return beta / np.sqrt(omab), 1.0 / np.sqrt(alpha), np.sqrt(beta)


def make_linear_schedule(steps: int, beta_start: float = 1e-4, beta_end: float = 0.02) -> NoiseSchedule:
    """diffusion.py:56-66."""
    if steps < 1:
        raise ValueError(f"steps must be >= 1, got {steps}")
    if steps == 1:
        return NoiseSchedule(np.array([beta_start], dtype=np.float64))
    return NoiseSchedule(np.linspace(beta_start, beta_end, steps, dtype=np.float64))
