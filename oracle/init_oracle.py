"""CPU restatement of the engine's deterministic parameter initialiser.

TEST INFRASTRUCTURE ONLY - imported by tests/, __graft_entry__.smoke() and the
bench cpu_baseline leg as the checker, never by the product path.

The reference has no parameter arithmetic at all (it is a schedule simulator,
SURVEY.md section 0), so the init is the engine's own definition: value_i =
mean + std*sqrt(3)*(u0+u1+u2+u3-2) with u_j = (splitmix64(seed + 4*(offset+i) + j)
>> 40) * 2^-24, summed left to right in fp32 with no fused multiply-add.  This
numpy version is bit-identical to ``zpp_init_param`` (csrc/kernels.cu).
"""

from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def init_values(n: int, seed: int, offset: int, mean: float, std: float) -> np.ndarray:
    idx = np.arange(n, dtype=np.uint64) + np.uint64(offset)
    with np.errstate(over="ignore"):
        base = np.uint64(seed) + np.uint64(4) * idx
    u = [(splitmix64(base + np.uint64(j)) >> np.uint64(40)).astype(np.float32)
         * np.float32(5.9604644775390625e-08) for j in range(4)]
    s = ((u[0] + u[1]) + u[2]) + u[3]
    s = s - np.float32(2.0)
    scale = np.float32(std) * np.float32(1.7320508075688772)
    return (np.float32(mean) + s * scale).astype(np.float32)
