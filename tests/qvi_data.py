"""Thermoforming data of the reference's QVI example (problems.py:210-235),
restated for the tests (the reference package is absent on the GPU box)."""
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ThermoformingData:
    load: float = 100.0
    gamma: float = 1.0

    @property
    def f(self):
        return self.load

    def xi(self, x, y):
        return np.sin(np.pi * x) * np.sin(np.pi * y)

    def mould(self, x, y):
        return (1.1 - 2.0 * np.maximum(np.abs(x - 0.5), np.abs(y - 0.5))
                + np.cos(8.0 * np.pi * x) * np.cos(8.0 * np.pi * y) / 10.0)

    def g(self, s):
        return np.clip((1.0 - np.asarray(s, dtype=float)) / 5.0, 0.0, 0.2)

    def g_deriv(self, s):
        s = np.asarray(s, dtype=float)
        return np.where((s >= 0.0) & (s <= 1.0), -0.2, 0.0)
