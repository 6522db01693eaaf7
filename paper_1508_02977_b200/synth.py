"""Seeded synthetic frame pairs for the five BASELINE.json configurations.

The reference's benchmark data (Middlebury RubberWhale, the paper's Highway/Wall scenes)
is not available; these generators stand in with the configured shapes, value ranges and
motion/illumination models (BASELINE.json ``configs``). Frames are fp64
gray levels on [0, 255]. Everything is numpy ``default_rng(seed)`` (PCG64), so
the oracle and the B200 build read identical bytes.

Frozen generator choices (recorded in BASELINE.md / DESIGN.md):
  c1  base 60 + 20 Gaussian blobs + 20 sin(2 pi x/16) sin(2 pi y/16); f2 = bilinear
      rotation by 2 deg about the centre (edge clamp) x (1 + 0.1 x/W); clipped.
  c2  1/f random-phase noise background; 2 ellipses + 1 rectangle with own noise textures
      translating by non-integer velocities (|v| <= 3 px); f2 x degree-2 random polynomial
      gain in [0.9, 1.1].
  c3  4-octave value noise warped by 8 Gaussian vortices (max 5 px) + additive offset in
      [-10, 10]; c4 = c3 generator with spatial scales x2 (max displacement kept at 5 px).
  c5  value-noise texture; flow (+3,0) / (-1,2) across a random smooth curve; gain 0.7 / 1.3
      across a second curve; + N(0, 2^2) per frame.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    H: int
    W: int
    sigma: float
    parts: int
    overlap: int
    n_passes: int
    tol: float = 1e-10
    seed: int = 0
    rho: float = 2.5
    alpha0: float = 1000.0
    lambda0: float = 1000.0
    kappa: float = 10.0
    eta_threshold: float = 0.1
    overlaps: tuple = field(default_factory=tuple)


CONFIGS = {
    "c1": Config("c1_128x128_2x2_ov4", 128, 128, 1.0, 4, 4, 3),
    "c2": Config("c2_388x584_4x4_ov2", 388, 584, 1.5, 16, 2, 5),
    "c3": Config("c3_1080x1920_8x8_ov4", 1080, 1920, 1.5, 64, 4, 10),
    "c4": Config("c4_2160x3840_16x16_ov4", 2160, 3840, 1.5, 256, 4, 10),
    "c5": Config("c5_1024x1024_4x4_ov1-8", 1024, 1024, 1.5, 16, 4, 8, overlaps=(1, 2, 4, 8)),
}


def _bilinear(img: np.ndarray, X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Bilinear sample with edge clamp."""
    H, W = img.shape
    X = np.clip(X, 0.0, W - 1.0)
    Y = np.clip(Y, 0.0, H - 1.0)
    x0 = np.minimum(np.floor(X).astype(np.int64), W - 2)
    y0 = np.minimum(np.floor(Y).astype(np.int64), H - 2)
    fx = X - x0
    fy = Y - y0
    a = img[y0, x0]
    b = img[y0, x0 + 1]
    c = img[y0 + 1, x0]
    d = img[y0 + 1, x0 + 1]
    return (a * (1 - fx) + b * fx) * (1 - fy) + (c * (1 - fx) + d * fx) * fy


def gen_c1(seed: int = 0, H: int = 128, W: int = 128):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)

    def f1_at(X, Y):
        v = np.full(X.shape, 60.0)
        for cx, cy, s, a in blobs:
            v += a * np.exp(-((X - cx) ** 2 + (Y - cy) ** 2) / (2 * s * s))
        v += 20.0 * np.sin(2 * np.pi * X / 16.0) * np.sin(2 * np.pi * Y / 16.0)
        return np.clip(v, 0.0, 255.0)

    blobs = [(rng.uniform(0, W), rng.uniform(0, H), rng.uniform(3, 12), rng.uniform(20, 120))
             for _ in range(20)]
    f1 = f1_at(xx, yy)
    c = np.array([(W - 1) / 2.0, (H - 1) / 2.0])
    th = np.deg2rad(2.0)
    # f2(x) = f1(R^-1 (x - c) + c): content rotates by +2 deg
    ct, st = np.cos(-th), np.sin(-th)
    Xs = ct * (xx - c[0]) - st * (yy - c[1]) + c[0]
    Ys = st * (xx - c[0]) + ct * (yy - c[1]) + c[1]
    f2 = np.clip(_bilinear(f1, Xs, Ys) * (1.0 + 0.1 * xx / W), 0.0, 255.0)
    ct2, st2 = np.cos(th), np.sin(th)
    u = ct2 * (xx - c[0]) - st2 * (yy - c[1]) + c[0] - xx
    v = st2 * (xx - c[0]) + ct2 * (yy - c[1]) + c[1] - yy
    return f1, f2, np.stack([u, v])


def _pink_noise(rng, H, W, beta=1.0):
    ky = np.fft.fftfreq(H)[:, None]
    kx = np.fft.rfftfreq(W)[None, :]
    k = np.sqrt(kx * kx + ky * ky)
    k[0, 0] = 1.0
    amp = 1.0 / k ** beta
    amp[0, 0] = 0.0
    amp[k > 0.25] = 0.0  # band limit
    ph = rng.uniform(0, 2 * np.pi, amp.shape)
    img = np.fft.irfft2(amp * np.exp(1j * ph), s=(H, W))
    img -= img.min()
    return img / img.max() * 255.0


def gen_c2(seed: int = 0, H: int = 388, W: int = 584):
    rng = np.random.default_rng(seed)
    bg = _pink_noise(rng, H, W)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    objs = []
    for kind in ("ellipse", "ellipse", "rect"):
        tex = _pink_noise(rng, H, W)
        cx, cy = rng.uniform(0.25 * W, 0.75 * W), rng.uniform(0.25 * H, 0.75 * H)
        ax, ay = rng.uniform(30, 90), rng.uniform(25, 70)
        ang = rng.uniform(0, 2 * np.pi)
        mag = rng.uniform(1.0, 3.0)
        vel = (mag * np.cos(ang), mag * np.sin(ang))
        objs.append((kind, tex, cx, cy, ax, ay, vel))

    def frame(t):
        img = bg.copy()
        flow = np.zeros((2, H, W))
        for kind, tex, cx, cy, ax, ay, (vx, vy) in objs:
            X, Y = xx - t * vx, yy - t * vy  # texture coordinates at time t
            if kind == "ellipse":
                inside = ((X - cx) / ax) ** 2 + ((Y - cy) / ay) ** 2 <= 1.0
            else:
                inside = (np.abs(X - cx) <= ax) & (np.abs(Y - cy) <= ay)
            img = np.where(inside, _bilinear(tex, X, Y), img)
            flow[0] = np.where(inside, vx, flow[0])
            flow[1] = np.where(inside, vy, flow[1])
        return img, flow

    f1, flow = frame(0.0)
    f2, _ = frame(1.0)
    cf = rng.uniform(-1, 1, 6)
    xn, yn = xx / W - 0.5, yy / H - 0.5
    poly = cf[0] + cf[1] * xn + cf[2] * yn + cf[3] * xn * xn + cf[4] * xn * yn + cf[5] * yn * yn
    poly = (poly - poly.min()) / max(poly.max() - poly.min(), 1e-12)
    f2 = np.clip(f2 * (0.9 + 0.2 * poly), 0.0, 255.0)
    return f1, f2, flow


def _value_noise_fn(rng, octaves, base_cell):
    """Multiscale value noise as a function of continuous (X, Y)."""
    grids = []
    for o in range(octaves):
        cell = base_cell / (2 ** o)
        grids.append((cell, rng.uniform(0, 1, (4096 // max(int(cell), 1) + 8,) * 2), 0.5 ** o))

    def f(X, Y):
        v = np.zeros(X.shape)
        tot = 0.0
        for cell, g, w in grids:
            gx = np.mod(X / cell, g.shape[1] - 2)
            gy = np.mod(Y / cell, g.shape[0] - 2)
            x0 = np.floor(gx).astype(np.int64)
            y0 = np.floor(gy).astype(np.int64)
            tx, ty = gx - x0, gy - y0
            tx = tx * tx * (3 - 2 * tx)
            ty = ty * ty * (3 - 2 * ty)
            a, b = g[y0, x0], g[y0, x0 + 1]
            c, d = g[y0 + 1, x0], g[y0 + 1, x0 + 1]
            v += w * ((a * (1 - tx) + b * tx) * (1 - ty) + (c * (1 - tx) + d * tx) * ty)
            tot += w
        return 255.0 * v / tot

    return f


def gen_c3(seed: int = 0, H: int = 1080, W: int = 1920, scale: float = 1.0):
    rng = np.random.default_rng(seed)
    noise = _value_noise_fn(rng, 4, 32.0 * scale)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    u = np.zeros((H, W))
    v = np.zeros((H, W))
    for _ in range(8):
        cx, cy = rng.uniform(0, W), rng.uniform(0, H)
        s = rng.uniform(80, 250) * scale
        sgn = rng.choice([-1.0, 1.0])
        g = np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))
        u += sgn * -(yy - cy) / s * g
        v += sgn * (xx - cx) / s * g
    mag = np.sqrt(u * u + v * v).max()
    u *= 5.0 / mag
    v *= 5.0 / mag
    f1 = noise(xx, yy)
    f2 = noise(xx - u, yy - v)
    ox, oy = rng.uniform(0, 2 * np.pi, 2)
    off = 10.0 * np.sin(2 * np.pi * xx / (W * 0.7) + ox) * np.cos(2 * np.pi * yy / (H * 0.9) + oy)
    f2 = f2 + off
    return f1, f2, np.stack([u, v])


def gen_c4(seed: int = 0):
    return gen_c3(seed, 2160, 3840, scale=2.0)


def gen_c5(seed: int = 0, H: int = 1024, W: int = 1024):
    rng = np.random.default_rng(seed)
    noise = _value_noise_fn(rng, 4, 24.0)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)

    def curve(rng):
        a = rng.uniform(-1, 1, 3)
        return (0.5 + 0.15 * a[0] * np.sin(2 * np.pi * xx / W * (1 + a[1])) + 0.1 * a[2]) * H

    c1 = curve(rng)
    c2 = curve(rng)
    region = yy < c1
    u = np.where(region, 3.0, -1.0)
    v = np.where(region, 0.0, 2.0)
    f1 = noise(xx, yy)
    f2 = noise(xx - u, yy - v)
    gain = np.where(xx + 0.3 * (yy - c2) < 0.5 * W, 0.7, 1.3)
    f2 = f2 * gain
    f1 = f1 + rng.normal(0, 2.0, f1.shape)
    f2 = f2 + rng.normal(0, 2.0, f2.shape)
    return f1, f2, np.stack([u, v])


GENERATORS = {"c1": gen_c1, "c2": gen_c2, "c3": gen_c3, "c4": gen_c4, "c5": gen_c5}


def make(name: str, seed: int | None = None):
    """(f0, f1, true_flow, Config) for configuration ``name``."""
    cfg = CONFIGS[name]
    f0, f1, flow = GENERATORS[name](cfg.seed if seed is None else seed)
    return (np.ascontiguousarray(f0, dtype=np.float64), np.ascontiguousarray(f1, dtype=np.float64),
            flow, cfg)
