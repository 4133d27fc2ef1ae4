"""Seeded synthetic scenes standing in for the paper's ECSSD images and
PoolNet saliency maps, which are not available here.

Rules (BASELINE.json configs):
  * generator: numpy Generator(PCG64(seed)); obj seed 1000 + 10 cfg + layer,
    mask seed 2000 + 10 cfg + layer;
  * object: sum of 8 Gaussian blobs, centres uniform in the object,
    sigma ~ U[4,16] * (No/128) px, peak ~ U[64,255]; pixels below the
    (1 - f)-quantile of the blob sum are zeroed (f = 0.30, or 0.15 for the
    multi-depth config) — the literal spec gives ~90% nonzero at 128^2, so
    this calibration is required; values rounded and
    clipped to uint8 and used AS-IS as amplitudes (no /255: keeps the DWT and
    A_eff exact in fp32);
  * saliency: PCG64 white noise smoothed by a periodic Gaussian of
    sigma = No/16 (FFT), thresholded at its (1 - f_s)-quantile into a binary
    {0, 255} uint8 mask (255 -> 1.0 under the u8 saliency scale), with exact
    empty and full masks at f_s = 0 and 1.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

WAVELENGTH = 532e-9


@dataclass
class SceneConfig:
    name: str
    cfg: int
    object_size: int
    plane_size: int
    pitch: float
    depths: tuple[float, ...]
    nonzero_frac: float = 0.30
    saliency_frac: float = 0.25
    method: str = "direct"
    wavelength: float = WAVELENGTH

    @property
    def n_layers(self) -> int:
        return len(self.depths)


CONFIGS = {
    0: SceneConfig("cfg0_128_direct", 0, 128, 128, 8e-6, (0.2,)),
    1: SceneConfig("cfg1_512on1024_direct", 1, 512, 1024, 8e-6, (0.2,)),
    2: SceneConfig("cfg2_1024on2048_lut", 2, 1024, 2048, 8e-6, (0.2,), method="lut"),
    3: SceneConfig("cfg3_4x1024on4096_multidepth", 3, 1024, 4096, 4e-6, (0.15, 0.20, 0.25, 0.30),
                   nonzero_frac=0.15),
    4: SceneConfig("cfg4_2048on4096_direct", 4, 2048, 4096, 4e-6, (0.2,)),
}


def blob_object(no: int, seed: int, nonzero_frac: float = 0.30) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    cx = rng.uniform(0, no, 8)
    cy = rng.uniform(0, no, 8)
    sigma = rng.uniform(4, 16, 8) * (no / 128.0)
    peak = rng.uniform(64, 255, 8)
    yy = np.arange(no, dtype=np.float64)[:, None]
    xx = np.arange(no, dtype=np.float64)[None, :]
    field = np.zeros((no, no))
    for i in range(8):
        field += peak[i] * np.exp(-((xx - cx[i]) ** 2 + (yy - cy[i]) ** 2) / (2 * sigma[i] ** 2))
    thr = np.quantile(field, 1.0 - nonzero_frac)
    obj = np.where(field >= thr, np.clip(np.rint(field), 0, 255), 0).astype(np.uint8)
    return obj


def smooth_mask(no: int, seed: int, frac: float) -> np.ndarray:
    """Binary uint8 mask {0,255}: top `frac` of a smoothed noise field."""
    if frac <= 0.0:
        return np.zeros((no, no), np.uint8)
    if frac >= 1.0:
        return np.full((no, no), 255, np.uint8)
    rng = np.random.Generator(np.random.PCG64(seed))
    noise = rng.standard_normal((no, no))
    sigma = no / 16.0
    f = np.fft.fftfreq(no)
    g = np.exp(-2 * (np.pi * sigma) ** 2 * (f[:, None] ** 2 + f[None, :] ** 2))
    smooth = np.real(np.fft.ifft2(np.fft.fft2(noise) * g))
    thr = np.quantile(smooth, 1.0 - frac)
    return np.where(smooth >= thr, 255, 0).astype(np.uint8)


@dataclass
class Scene:
    config: SceneConfig
    objects: np.ndarray  # (L, No, No) uint8
    masks: np.ndarray    # (L, No, No) uint8 {0,255}
    extra: dict = field(default_factory=dict)


def make_scene(cfg: int | SceneConfig, saliency_frac: float | None = None,
               object_size: int | None = None, plane_size: int | None = None) -> Scene:
    c = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if object_size is not None or plane_size is not None or saliency_frac is not None:
        c = SceneConfig(**{**c.__dict__})
        if object_size is not None:
            c.object_size = object_size
        if plane_size is not None:
            c.plane_size = plane_size
        if saliency_frac is not None:
            c.saliency_frac = saliency_frac
    objs, masks = [], []
    for layer in range(c.n_layers):
        objs.append(blob_object(c.object_size, 1000 + 10 * c.cfg + layer, c.nonzero_frac))
        mseed = 2000 + 10 * c.cfg + (0 if c.cfg == 4 else layer)
        masks.append(smooth_mask(c.object_size, mseed, c.saliency_frac))
    return Scene(c, np.stack(objs), np.stack(masks))


def scene_digest(scene: Scene) -> dict:
    """SHA-256 of the object and mask bytes plus the realised fractions, so
    the CPU oracle, the GPU box and the committed fixtures can be shown to use
    byte-identical inputs (tests/golden/scene_digests.json)."""
    o, m = np.ascontiguousarray(scene.objects), np.ascontiguousarray(scene.masks)
    return {
        "objects_sha256": hashlib.sha256(o.tobytes()).hexdigest(),
        "masks_sha256": hashlib.sha256(m.tobytes()).hexdigest(),
        "shape": list(o.shape),
        "nonzero_frac": float(np.count_nonzero(o) / o.size),
        "salient_frac": float(np.count_nonzero(m) / m.size),
    }


def digest_cases() -> list[tuple[str, int, float | None]]:
    """(name, cfg, saliency_frac) of every BASELINE config, cfg4 per sweep point."""
    cases = [(CONFIGS[c].name, c, None) for c in (0, 1, 2, 3)]
    cases += [(f"{CONFIGS[4].name}_sal{f:.2f}", 4, f) for f in (0.0, 0.10, 0.25, 0.50, 1.0)]
    return cases
