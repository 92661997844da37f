"""The published parameter sets (presets.py:19-69 of the reference) as data.

Same prime pool, plaintext moduli, preset ids and prime-count rule
(round(log q / 30) primes of the pool) as the reference, so that contexts built
here have the reference's fingerprints.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import bfv as B
from .errors import UnsupportedParametersError

RNS_PRIME_POOL = (
    1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641,
    1071513601, 1071415297, 1071087617, 1070727169, 1070432257, 1069219841,
)
MNIST_T = 5522259017729
CIFAR_T = (2424833, 2654209, 2752513, 3604481, 3735553,
           4423681, 4620289, 4816897, 4882433, 5308417)


@dataclass(frozen=True)
class Preset:
    id: str
    ring_degree: int
    log_q: int
    plaintext_moduli: tuple
    depth: int
    security_bits: int
    security_class: str
    rns_primes: tuple

    @property
    def channels(self) -> int:
        return len(self.plaintext_moduli)


def _preset(pid, n, log_q, moduli, depth, lam, sec="paper"):
    return Preset(pid, n, log_q, tuple(moduli), depth, lam, sec, RNS_PRIME_POOL[: round(log_q / 30)])


PRESETS = {
    "toy": _preset("toy", 1 << 12, 180, [MNIST_T], 4, 0, "toy-insecure"),
    "1": _preset("1", 1 << 13, 330, [MNIST_T], 4, 82),
    "2": _preset("2", 1 << 13, 360, [MNIST_T], 5, 76),
    "3": _preset("3", 1 << 14, 330, [MNIST_T], 4, 175),
    "4": _preset("4", 1 << 14, 360, [MNIST_T], 5, 159),
    "5": _preset("5", 1 << 13, 300, CIFAR_T, 7, 91),
}

_CTX: dict = {}


def load_preset(pid) -> Preset:
    if str(pid) not in PRESETS:
        raise UnsupportedParametersError(f"unknown preset '{pid}' (have: {', '.join(sorted(PRESETS))})")
    return PRESETS[str(pid)]


def build_context(preset: Preset, t_index: int = 0, relin_base: int = 1 << 16) -> B.BfvParams:
    """BfvParams for one plaintext channel (presets.py:145-162)."""
    if not 0 <= t_index < preset.channels:
        raise UnsupportedParametersError(f"channel {t_index} out of range for preset {preset.id}")
    key = (preset.ring_degree, preset.rns_primes)
    ctx = _CTX.get(key)
    if ctx is None:
        ctx = B.RnsContext(preset.ring_degree, list(preset.rns_primes))
        _CTX[key] = ctx
    return B.BfvParams(ctx, preset.plaintext_moduli[t_index], relin_base=relin_base,
                       depth=preset.depth, security_bits=preset.security_bits)
