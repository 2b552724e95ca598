"""Counter-based RNG in plain torch integer ops (CPU and CUDA give identical bits).

u = hash(seed, image, stream, counter) -> 24-bit uniform in (0, 1).  All products
are done on 16-bit halves so no int64 intermediate overflows.
"""
from __future__ import annotations

import math

import torch

_M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    lo, hi = c & 0xFFFF, (c >> 16) & 0xFFFF
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _M32


def _hash32(x: torch.Tensor) -> torch.Tensor:
    # "triple32"-style integer finaliser (xor-shift / multiply), all in [0, 2^32)
    x = x & _M32
    x = x ^ (x >> 17)
    x = _mul32(x, 0xED5AD4BB)
    x = x ^ (x >> 11)
    x = _mul32(x, 0xAC4C1B51)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x31848BAB)
    x = x ^ (x >> 14)
    return x


def _key(seed: int, image: torch.Tensor, stream: int, counter: torch.Tensor) -> torch.Tensor:
    h = _hash32(image * 0x9E37 + (seed & 0xFFFF) * 0x10001 + stream * 0x3C6EF)
    h = _hash32(h ^ (_hash32(counter + 0x632BE5AB) + stream))
    return _hash32(h + (seed >> 16))


def uniform01(seed: int, image: torch.Tensor, stream: int, counter: torch.Tensor,
              dtype=torch.float64) -> torch.Tensor:
    """Uniform in (0,1): ((h >> 8) + 0.5) / 2^24.  image/counter broadcast (int64 tensors)."""
    h = _key(seed, image.to(torch.int64), stream, counter.to(torch.int64))
    return (((h >> 8).to(dtype)) + 0.5) * (1.0 / 16777216.0)


def normal01(seed: int, image: torch.Tensor, stream: int, counter: torch.Tensor,
             dtype=torch.float64) -> torch.Tensor:
    """Standard normal by Box-Muller from two counter-keyed uniforms."""
    c = counter.to(torch.int64) * 2
    u1 = uniform01(seed, image, stream, c, torch.float64)
    u2 = uniform01(seed, image, stream, c + 1, torch.float64)
    z = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)
    return z.to(dtype)
