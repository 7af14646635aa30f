"""Synthetic moving-rectangle clips: the reference's only video source.

Host-side restatement of the *input generator* (synth.hpp:45-101) plus the
benchmark recipes C1-C5 of SURVEY.md §8(d).  The host computes each shape's
integer top-left corner per frame with the reference's exact expression
``lround(x0 + vx * t)`` (synth.hpp:307-314); the device rasteriser
(``trb_synth_raster``) paints the frames, later shapes overwriting earlier
ones (synth.hpp:317-328).  Generation is never inside a timed region.

Recipe parameters are drawn from ``Rng(shape_seed)`` (rng.hpp:12-51, a
restated mt19937_64): per shape, in this order, ``w, h = uniform_int(smin,
smax)``, ``color = uniform_int(96, 255)``, then ``x0, y0, x1, y1`` uniform
over the positions that keep the largest shape inside the frame.  In a
"crossing" recipe every odd shape runs the previous shape's path in reverse
(its own endpoints are still drawn, then replaced), so paths overlap and
blobs occlude and merge.  Velocities are endpoint-derived, hence
``n_frames`` is part of the recipe.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

_M64 = (1 << 64) - 1


class Rng:
    """mt19937_64 + the reference's hand-rolled draws (rng.hpp:12-51)."""

    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _M64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt = mt
        self._idx = 312
        self._spare = 0.0
        self._have_spare = False

    def next_u64(self) -> int:
        mt = self._mt
        if self._idx >= 312:
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self._idx = 0
        y = mt[self._idx]
        self._idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y &= _M64
        y ^= y >> 43
        return y

    def uniform(self, lo: Optional[float] = None, hi: Optional[float] = None) -> float:
        u = float(self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_int(self, lo: int, hi: int) -> int:
        span = ((hi - lo) & _M64) + 1
        return lo + (self.next_u64() % span)

    def gaussian(self, mean: float = 0.0, sigma: float = 1.0) -> float:
        if self._have_spare:
            self._have_spare = False
            g = self._spare
        else:
            u1 = self.uniform()
            while u1 <= 0.0:
                u1 = self.uniform()
            u2 = self.uniform()
            r = math.sqrt(-2.0 * math.log(u1))
            a = 2.0 * 3.14159265358979323846 * u2
            self._spare = r * math.sin(a)
            self._have_spare = True
            g = r * math.cos(a)
        return mean + sigma * g


def mix_seed(seed: int, salt: int) -> int:
    """rng.hpp:63-68"""
    z = (seed + 0x9E3779B97F4A7C15 * (salt + 1)) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def lround(x: float) -> int:
    """std::lround: round half away from zero, exact for doubles."""
    if x < 0:
        return -lround(-x)
    f = math.floor(x)
    return int(f) + (1 if x - f >= 0.5 else 0)


@dataclass
class Shape:
    """ShapeSpec (synth.hpp:16-25)."""
    width: int
    height: int
    color: Tuple[int, int, int]
    x0: float
    y0: float
    vx: float
    vy: float
    jitter_sigma: float = 0.0


@dataclass
class Clip:
    """ClipSpec (synth.hpp:27-33) + frame count and generator seed."""
    width: int
    height: int
    channels: int
    background: int
    shapes: List[Shape]
    n_frames: int
    seed: int = 0
    name: str = ""

    def rects(self, t: int, rng: Optional[Rng] = None) -> List[Tuple[int, int, int, int]]:
        """Integer (ix, iy, w, h) of every shape at frame t (synth.hpp:306-316).

        With jitter the draws must be consumed frame by frame through one
        ``rng`` (use :meth:`all_rects`)."""
        out = []
        for s in self.shapes:
            x = s.x0 + s.vx * t
            y = s.y0 + s.vy * t
            if s.jitter_sigma > 0.0:
                if rng is None:
                    raise ValueError("jittered clips need the shared Rng; use all_rects()")
                x += rng.gaussian(0.0, s.jitter_sigma)
                y += rng.gaussian(0.0, s.jitter_sigma)
            ix, iy = lround(x), lround(y)
            if ix < 0 or iy < 0 or ix + s.width > self.width or iy + s.height > self.height:
                raise ValueError(f"shape leaves frame bounds at frame {t}")
            out.append((ix, iy, s.width, s.height))
        return out

    def all_rects(self, n: Optional[int] = None) -> List[List[Tuple[int, int, int, int]]]:
        rng = Rng(self.seed)
        return [self.rects(t, rng) for t in range(self.n_frames if n is None else n)]

    def colors(self) -> List[Tuple[int, int, int]]:
        return [s.color for s in self.shapes]

    def shape_arrays(self):
        """(int32 n*5, float64 n*5) packing used by the C ABIs."""
        si, sd = [], []
        for s in self.shapes:
            si += [s.width, s.height, s.color[0], s.color[1], s.color[2]]
            sd += [s.x0, s.y0, s.vx, s.vy, s.jitter_sigma]
        return si, sd


def random_clip(width: int, height: int, n_shapes: int, smin: int, smax: int, crossing: bool, shape_seed: int,
                synth_seed: int, n_frames: int = 300, background: int = 16, name: str = "") -> Clip:
    rng = Rng(shape_seed)
    span = n_frames - 1
    shapes: List[Shape] = []
    paths = []
    for k in range(n_shapes):
        w = rng.uniform_int(smin, smax)
        h = rng.uniform_int(smin, smax)
        c = rng.uniform_int(96, 255)
        x0 = rng.uniform(0.0, float(width - smax - 1))
        y0 = rng.uniform(0.0, float(height - smax - 1))
        x1 = rng.uniform(0.0, float(width - smax - 1))
        y1 = rng.uniform(0.0, float(height - smax - 1))
        if crossing and k % 2 == 1:
            px0, py0, px1, py1 = paths[k - 1]
            x0, y0, x1, y1 = px1, py1, px0, py0
        paths.append((x0, y0, x1, y1))
        shapes.append(Shape(w, h, (c, c, c), x0, y0, (x1 - x0) / span, (y1 - y0) / span))
    return Clip(width, height, 1, background, shapes, n_frames, synth_seed, name)


def recipe(name: str, stream: int = 0, n_frames: int = 300) -> Clip:
    """SURVEY.md §8(d) recipes C1-C5 (C5 = stream `stream` of 64 x C3)."""
    if name == "C1":
        return random_clip(320, 240, 3, 12, 20, False, 1, 1001, n_frames, name="C1")
    if name == "C2":
        span = n_frames - 1
        ox = [0, -30, 30, -60, 60, -90, 90, 0]
        oy = [0, 40, 40, 80, 80, 120, 120, 160]
        shapes = []
        for i in range(8):
            v = 220 if i % 2 == 0 else 30
            shapes.append(Shape(12, 28, (v, v, v), 200.0 + ox[i], 60.0 + oy[i], 240.0 / span, 200.0 / span))
        return Clip(640, 480, 1, 90, shapes, n_frames, 1002, "C2")
    if name == "C3":
        return random_clip(1920, 1080, 20, 40, 80, True, 3, 1003, n_frames, name="C3")
    if name == "C4":
        return random_clip(3840, 2160, 50, 48, 96, True, 4, 1004, n_frames, name="C4")
    if name == "C5":
        return random_clip(1920, 1080, 20, 40, 80, True, mix_seed(3, stream), mix_seed(1003, stream), n_frames,
                           name=f"C5[{stream}]")
    raise ValueError(f"unknown recipe {name!r}")


def harness_vision_clip() -> Clip:
    """The harness_test vision clip (harness_test.cpp:377-389): 48x36 RGB,
    W=9 window, 29 frames, seed 4321."""
    n = 9 + 20
    span = n - 1
    shapes = [Shape(7, 7, (220, 60, 40), 3.0, 3.0, (28.0 - 3.0) / span, (20.0 - 3.0) / span),
              Shape(6, 6, (40, 80, 230), 38.0, 26.0, (4.0 - 38.0) / span, (6.0 - 26.0) / span)]
    return Clip(48, 36, 3, 0, shapes, n, 4321, "harness_vision")


def bench_vision_clip(window: int = 91, seed: int = 0) -> Clip:
    """bench_run's transparency clip (harness.hpp:571-581): 96x72 RGB,
    window+60 frames, seed mix_seed(cfg.seed, stable_hash("bench/clip"))."""
    n = window + 60
    span = n - 1
    shapes = [Shape(9, 9, (220, 60, 40), 4.0, 8.0, (83.0 - 4.0) / span, (53.0 - 8.0) / span),
              Shape(8, 8, (40, 80, 230), 84.0, 56.0, (6.0 - 84.0) / span, (10.0 - 56.0) / span)]
    return Clip(96, 72, 3, 0, shapes, n, mix_seed(seed, stable_hash("bench/clip")), "bench_vision")


def stable_hash(s: str) -> int:
    """FNV-1a, rng.hpp:54-61"""
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & _M64
    return h


def raster_host(clip: Clip, rects: Sequence[Tuple[int, int, int, int]]):
    """numpy raster of one frame from integer rects (for tests / host e2e)."""
    import numpy as np
    f = np.full((clip.height, clip.width, clip.channels), clip.background, dtype=np.uint8)
    for (ix, iy, w, h), s in zip(rects, clip.shapes):
        f[iy:iy + h, ix:ix + w, :] = np.array(s.color[:clip.channels] if clip.channels == 3 else s.color[:1],
                                              dtype=np.uint8)
    return f.reshape(-1) if clip.channels == 1 else f.reshape(-1)


def device_frames(clips: Sequence[Clip], n_frames: int, cuda_stream: int = 0, device=None):
    """Frames 0..n_frames-1 of every clip rasterised on the device (one
    launch per clip): a uint8 tensor [S, n_frames, w*h*ch].  The integer
    rects come from Clip.rects (synth.hpp:307-314's lround on the host); the
    device only paints them (later shapes overwrite earlier ones).  This is
    the bench's input path; tests hash it against the reference synth."""
    import torch
    from . import api
    c0 = clips[0]
    fb = c0.width * c0.height * c0.channels
    buf = torch.empty((len(clips), n_frames, fb), dtype=torch.uint8, device=device or "cuda")
    for s, c in enumerate(clips):
        rects = [c.rects(t) for t in range(n_frames)]
        api.synth_raster_frames(buf[s, 0].data_ptr(), fb, c.width, c.height, c.channels, c.background, rects,
                                c.colors(), cuda_stream)
    torch.cuda.synchronize()
    return buf
