"""Deterministic synthetic workloads for the BASELINE configs.

The reference has no float volumes and no Kingsnake / Rayleigh-Taylor /
Richtmyer-Meshkov data (the paper's datasets are not available offline), so
these generators define the configs:

  C1  blobs(64)   64^3 f32 Gaussian blobs, 128x128, n_sg 20, render at 15 deg
  C2  blobs(256)  256^3 f32, 512x512, n_sg 20
  C3  kingsnake() 1024x1024x795 u8, 1920x1080, n_sg 20 (the bench workload)
  C4  rt_like()   1024^3 f32, 1920x1080, n_sg 30, sweep 0-30 deg
  C5  rm_like()   2048x2048x1920 u8 (built on the GPU), 3840x2160, n_sg 40

Cameras follow the reference's sweep convention (bench.py:28-41 ==
synth.py:89-100): orbit about the volume centre, fov 45 deg, near = 0.15 r,
far = r + 2 * half_diag; "fill" cameras use r = 1.6 * max(size).
The sphere / bands presets reproduce synth.py:25-58 for the parity fixtures.
"""

from __future__ import annotations

import math

import numpy as np

from .camera import orbit_camera
from .volume import TransferFunction, Volume, make_volume

SPHERE_TF = ((0.0, 0.0, 0.0, 0.0, 0.0), (0.2, 0.0, 0.0, 0.0, 0.0),
             (0.47, 0.2, 0.4, 0.9, 0.35), (0.86, 0.9, 0.6, 0.2, 0.8),
             (1.0, 1.0, 0.8, 0.3, 0.9))
BANDS_TF = ((0.0, 0.0, 0.0, 0.0, 0.0), (0.15, 0.1, 0.2, 0.8, 0.25),
            (0.5, 0.2, 0.9, 0.3, 0.5), (1.0, 1.0, 0.3, 0.2, 0.85))
KINGSNAKE_TF = ((0.0, 0, 0, 0, 0), (0.12, 0, 0, 0, 0), (0.2, .8, .7, .5, .05),
                (0.55, .9, .5, .2, .6), (0.8, 1, 1, .9, .3), (1.0, 1, 1, 1, .4))
RT_TF = ((0.0, 0, 0, 0, 0), (0.3, .1, .2, .8, .02), (0.6, .9, .6, .2, .15),
         (1.0, 1, .2, .1, .5))
RM_TF = ((0.0, 0, 0, 0, 0), (0.22, 0, 0, 0, 0), (0.3, .9, .4, .1, .03),
         (0.55, .3, .7, .9, .12), (0.8, 1, .9, .6, .35), (1.0, 1, 1, 1, .6))


def blobs(n: int, k: int = 12, seed: int = 0) -> Volume:
    """Sum of K Gaussian blobs on [0,1]^3, clipped to [0,1], f32 (z, y, x)."""
    rng = np.random.default_rng(seed)
    c = (np.arange(n, dtype=np.float64) + 0.5) / n
    v = np.zeros((n, n, n), dtype=np.float64)
    for _ in range(k):
        centre = rng.uniform(0.2, 0.8, 3)
        sigma = rng.uniform(0.05, 0.15)
        amp = rng.uniform(0.4, 1.0)
        g = [np.exp(-((c - centre[a]) ** 2) / (2.0 * sigma * sigma)) for a in range(3)]
        v += amp * (g[2][:, None, None] * g[1][None, :, None]) * g[0][None, None, :]
    data = np.clip(v, 0.0, 1.0).astype(np.float32)
    return make_volume(data, "f32")


def kingsnake(dims=(1024, 1024, 795), seed: int = 1) -> Volume:
    """Kingsnake-shaped u8 volume: ellipsoid shell (200), faint interior (40),
    a coiled tube (150), integer jitter U{0..12} on non-zero voxels."""
    nx, ny, nz = dims
    ux = (np.arange(nx, dtype=np.float32) + 0.5) / nx
    uy = (np.arange(ny, dtype=np.float32) + 0.5) / ny
    uz = (np.arange(nz, dtype=np.float32) + 0.5) / nz
    X = ux[None, :] - 0.5
    Y = uy[:, None] - 0.5
    exy = (X / 0.46) ** 2 + (Y / 0.40) ** 2                      # (ny, nx)
    r = np.sqrt(X * X + Y * Y)
    ring = np.abs(r - 0.22) < 0.035
    ring_idx = np.nonzero(ring)
    phi = np.arctan2(Y, X)[ring_idx]                              # helix angle
    ring_dr2 = ((r[ring_idx] - 0.22) ** 2).astype(np.float32)
    pitch, turns, zc = 0.12, 3.0, 0.5
    z0 = zc - 0.5 * turns * pitch
    rng = np.random.default_rng(seed)
    data = np.zeros((nz, ny, nx), dtype=np.uint8)
    for iz in range(nz):
        e = exy + ((uz[iz] - 0.5) / 0.46) ** 2
        sl = np.zeros((ny, nx), dtype=np.uint8)
        sl[e < 1.0] = 40
        sl[(e >= 0.93) & (e < 1.0)] = 200
        # nearest helix pass over this angle: z = z0 + pitch * (phi/2pi + m)
        t = (uz[iz] - z0) / pitch - phi / (2.0 * math.pi)
        m = np.clip(np.rint(t), 0, turns - 1)
        zh = z0 + pitch * (phi / (2.0 * math.pi) + m)
        tube = (ring_dr2 + (uz[iz] - zh) ** 2) < 0.035 ** 2
        sub = sl[ring_idx]
        sub[tube] = 150
        sl[ring_idx] = sub
        nzm = sl > 0
        jit = rng.integers(0, 13, size=int(nzm.sum()), dtype=np.uint8)
        sl[nzm] = np.minimum(255, sl[nzm].astype(np.int16) + jit).astype(np.uint8)
        data[iz] = sl
    return make_volume(data, "u8")


def rt_like(n: int = 1024, seed: int = 2) -> Volume:
    """Rayleigh-Taylor-shaped f32 volume: a perturbed
    heavy/light interface z = h(x, y) = 0.5 + sum_m A_m sin(2 pi k_m . (x, y) +
    phi_m) (16 integer wave vectors, |k| in [2, 16], A ~ 1/|k|, sum A = 0.12),
    density rho = 0.5 - 0.5 tanh((z - h) / 0.02), plus 3-octave separable
    sinusoidal noise of amplitude 0.05 within |z - h| < 0.1, clipped to [0, 1]."""
    rng = np.random.default_rng(seed)
    ks = []
    while len(ks) < 16:
        k = rng.integers(-16, 17, size=2)
        if 2 <= np.hypot(*k) <= 16:
            ks.append(k)
    ks = np.array(ks, dtype=np.float64)
    amp = 1.0 / np.hypot(ks[:, 0], ks[:, 1])
    amp *= 0.12 / amp.sum()
    phi = rng.uniform(0, 2 * np.pi, 16)
    u = (np.arange(n, dtype=np.float64) + 0.5) / n
    X, Y = np.meshgrid(u, u, indexing="xy")  # (ny, nx)
    h = 0.5 + sum(amp[m] * np.sin(2 * np.pi * (ks[m, 0] * X + ks[m, 1] * Y) + phi[m])
                  for m in range(16))
    octs = [(4.0 * 2 ** o, 0.05 / 2 ** o, rng.uniform(0, 2 * np.pi, 3)) for o in range(3)]
    sx = [np.sin(2 * np.pi * f * u + p[0])[None, :] for f, _, p in octs]
    sy = [np.sin(2 * np.pi * f * u + p[1])[:, None] for f, _, p in octs]
    sxy = [(a * sx[i] * sy[i]).astype(np.float32) for i, (f, a, p) in enumerate(octs)]
    h32 = h.astype(np.float32)
    data = np.empty((n, n, n), dtype=np.float32)
    for iz in range(n):
        z = np.float32(u[iz])
        dz = z - h32
        rho = np.float32(0.5) - np.float32(0.5) * np.tanh(dz / np.float32(0.02))
        noise = sum(sxy[i] * np.float32(np.sin(2 * np.pi * f * u[iz] + p[2]))
                    for i, (f, a, p) in enumerate(octs))
        rho = np.where(np.abs(dz) < np.float32(0.1), rho + noise, rho)
        data[iz] = np.clip(rho, 0.0, 1.0)
    return make_volume(data, "f32")


def rm_modes(seed: int = 3) -> np.ndarray:
    """12 interface modes (kx, ky, amplitude, phase) of rm_like: integer wave
    vectors with |k| in [1, 12], A ~ |k|^-1.2 normalised to sum 0.1."""
    rng = np.random.default_rng(seed)
    ks = []
    while len(ks) < 12:
        k = rng.integers(-12, 13, size=2)
        if 1 <= np.hypot(*k) <= 12:
            ks.append(k)
    ks = np.array(ks, dtype=np.float64)
    amp = np.hypot(ks[:, 0], ks[:, 1]) ** -1.2
    amp *= 0.1 / amp.sum()
    phase = rng.uniform(0, 2 * np.pi, 12)
    return np.ascontiguousarray(np.stack([ks[:, 0], ks[:, 1], amp, phase], 1), np.float32)


def rm_like(dims=(2048, 2048, 1920), seed: int = 3, box=None):
    """Richtmyer-Meshkov-shaped u8 volume, synthesised on
    the device (vdi_synth_rm_u8): a mixing band of half-width 0.15 around a
    12-mode perturbed interface z = h(x, y), filled with 4-octave value-noise
    fbm mapped to 60..255; 0 outside. Returns a DeviceVolume; with box =
    (origin, size) only that resident box is synthesised (a DeviceVolume of
    the full dims holding a sub-box, as one rank of a bricked volume)."""
    import ctypes
    from . import _capi
    from . import device as dv
    from .volume import DeviceVolume
    t = dv.require_cuda()
    nx, ny, nz = dims
    if box is None:
        org, size = (0, 0, 0), (nx, ny, nz)
    else:
        org, size = tuple(int(v) for v in box[0]), tuple(int(v) for v in box[1])
    out = t.empty((size[2], size[1], size[0]), dtype=t.uint8, device="cuda")
    modes = rm_modes(seed)
    bx = np.array([*org, *size], np.int32)
    _capi.check(_capi.load().vdi_synth_rm_u8(
        dv.ptr(out), nx, ny, nz, bx.ctypes.data_as(ctypes.c_void_p),
        modes.ctypes.data_as(ctypes.c_void_p), ctypes.c_float(0.15), seed, dv.stream_handle()))
    t.cuda.current_stream().synchronize()
    return DeviceVolume(out, "u8", full_dims=dims if box is not None else None, origin=org)


def preset_volume(preset: str, dims: int = 128) -> Volume:
    """The reference's sphere / bands presets (synth.py:25-58), u8."""
    c1 = np.arange(dims, dtype=np.float64) + 0.5
    z, y, x = np.meshgrid(c1, c1, c1, indexing="ij")
    c = dims / 2.0
    if preset == "sphere":
        data = np.zeros((dims,) * 3, dtype=np.uint8)
        r = np.sqrt((x - c) ** 2 + (y - c) ** 2 + (z - c) ** 2)
        data[r < 0.35 * dims] = 120
        data[r < 0.18 * dims] = 220
    elif preset == "bands":
        band = (z // (dims / 8.0)).astype(np.int64) % 8
        levels = np.array([0, 220, 60, 160, 110, 240, 30, 190], dtype=np.uint8)
        data = levels[band]
    else:
        raise ValueError(f"unknown preset {preset!r}")
    return make_volume(data, "u8")


def preset_tf(preset: str) -> TransferFunction:
    table = {"sphere": SPHERE_TF, "blobs": SPHERE_TF, "bands": BANDS_TF,
             "kingsnake": KINGSNAKE_TF, "rt": RT_TF, "rm": RM_TF}
    return TransferFunction(table[preset])


def sweep_camera(vol: Volume, azimuth_deg: float, viewport,
                 radius_scale: float = 2.8, elevation_deg: float = 0.0):
    """Orbit camera about the volume centre (reference bench.py:28-41)."""
    size = vol.world_size
    center = size / 2.0
    radius = radius_scale * float(size.max())
    half_diag = 0.5 * float(np.linalg.norm(size))
    return orbit_camera(center, radius, azimuth_deg, elevation_deg,
                        fov_y=math.radians(45.0), near=0.15 * radius,
                        far=radius + 2.0 * half_diag, viewport=tuple(viewport))


CONFIGS = {
    # name: (volume factory, tf preset, viewport, n_sg, radius scale, render deg)
    "C1": (lambda: blobs(64), "blobs", (128, 128), 20, 2.8, 15.0),
    "C2": (lambda: blobs(256), "blobs", (512, 512), 20, 2.8, 15.0),
    "C3": (lambda: kingsnake(), "kingsnake", (1920, 1080), 20, 1.6, 15.0),
    "C4": (lambda: rt_like(), "rt", (1920, 1080), 30, 1.6, 15.0),
    "C5": (lambda: rm_like(), "rm", (3840, 2160), 40, 1.6, 15.0),
}


def config(name: str):
    """(vol, tf, gen_cam, render_cam, n_sg) for a BASELINE config."""
    make, tfp, vp, n_sg, rs, deg = CONFIGS[name]
    vol = make()
    tf = preset_tf(tfp)
    return (vol, tf, sweep_camera(vol, 0.0, vp, rs), sweep_camera(vol, deg, vp, rs),
            n_sg)
