"""The boundary reads the CALLER's LUTs.

The reference's apply_block / synthesize_base / refine / synthesize_progressive
superpose the FringeLut samples they are given (lut.support(),
synthesis.cpp:18-42,149-178,180-253), e.g. LUTs loaded from the f32 CGHL
cache (pipeline.cpp:174-177). Here those samples go to the device once
(wcgh_lut_create / stages.DeviceLut / FringeLut.device()) and are what the
GPU superposes; stage calls can accumulate into a device-resident plane
(wcgh_plane / stages.DevicePlane). A single perturbed LUT sample must change
the GPU result exactly as it changes the reference's (oracle/_ref, the
unmodified reference sources built by oracle/Makefile)."""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_2211_09938_b200 import _lib, stages
from paper_2211_09938_b200 import wavecgh as W
from paper_2211_09938_b200.hologram import HologramJob, JobSpec

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref absent")

WL, PITCH, Z = 532e-9, 8e-6, 0.1  # ref_random_n16/n32 geometry (test_synthesis.cpp:17)


def _perturbed(sup, iy, ix, delta):
    s = np.array(sup, np.complex128, copy=True)
    s[iy, ix] += delta
    return s


def test_device_lut_upload_download_and_validation(ctx):
    g = golden("ref_random_n16")
    for b in (1, 2, 4, 8):
        lut = stages.DeviceLut((WL, PITCH, Z), 16, b, g[f"lut{b}"])
        assert np.array_equal(lut.download(), g[f"lut{b}"].astype(np.complex64))
        lut32 = stages.DeviceLut((WL, PITCH, Z), 16, b, g[f"lut{b}"].astype(np.complex64))
        assert np.array_equal(lut32.download(), lut.download())
    built = stages.DeviceLut((WL, PITCH, Z), 16, 2)  # samples=None: built on the device
    assert np.abs(built.download() - g["lut2"]).max() / np.abs(g["lut2"]).max() <= 2e-7
    bad = g["lut1"].copy()
    bad[3, 4] = np.nan
    with pytest.raises(_lib.ValidationError):
        stages.DeviceLut((WL, PITCH, Z), 16, 1, bad)
    with pytest.raises(_lib.ValidationError):
        stages.DeviceLut((WL, PITCH, Z), 16, 3, g["lut1"])
    with pytest.raises(_lib.ValidationError):
        stages.DeviceLut((WL, PITCH, Z), 16, 1, g["lut1"][:-1])


@needs_ref
@pytest.mark.parametrize("block", [1, 2, 4, 8])
def test_perturbed_lut_sample_changes_apply_block_like_reference(ctx, block):
    g = golden("ref_random_n16")
    n = 16
    sup = g[f"lut{block}"]
    cx = cy = (n // block) // 2
    # perturb the sample that lands on pixel (x, y) = (cx*B + 3, cy*B - 2)
    dx, dy = 3 - 0, -2
    iy, ix = dy + n - 1, dx + n - 1
    delta = 0.37 - 0.21j
    w = 0.7 - 0.3j
    base_plane = (np.random.default_rng(3).standard_normal((n, n, 2)) @ [1, 1j]) * 1e-3
    pert = _perturbed(sup, iy, ix, delta)
    ref0, ops0 = O.ref_apply_block_lut(base_plane, sup, WL, PITCH, Z, block, cx, cy, w)
    ref1, ops1 = O.ref_apply_block_lut(base_plane, pert, WL, PITCH, Z, block, cx, cy, w)
    assert ops0 == ops1 == 1
    got = []
    for s in (sup, pert):
        lut = stages.DeviceLut((WL, PITCH, Z), n, block, s)
        plane = stages.DevicePlane(n).upload(base_plane)
        ops = lut.apply_blocks(plane, [cy * (n // block) + cx], [w.real], [w.imag])
        assert ops == 1
        got.append(plane.download(np.complex128))
    assert O.max_rel_error(got[0], ref0) <= 1e-6
    assert O.max_rel_error(got[1], ref1) <= 1e-6
    d_ref, d_gpu = ref1 - ref0, got[1] - got[0]
    y, x = cy * block + dy, cx * block + dx
    assert np.count_nonzero(d_ref) == 1 and d_ref[y, x] != 0  # the reference: one pixel moves by w*delta
    assert abs(d_ref[y, x] - w * delta) <= 1e-12
    nz = np.argwhere(d_gpu != 0)
    assert nz.tolist() == [[y, x]], nz  # ours: the same pixel, nothing else
    # complex64 LUT samples: the two planes differ by w*(S+delta) - w*S, each
    # rounded once to fp32 at the sample's magnitude
    assert abs(d_gpu[y, x] - w * delta) <= 4e-7 * abs(w) * abs(pert[iy, ix]) + 1e-7


@needs_ref
def test_mirror_apply_block_and_refine_read_the_caller_lut(ctx):
    """wavecgh.apply_block / refine / synthesize_base with a FringeLut whose
    samples the caller changed: numpy planes (host add) and DevicePlane
    (resident) both follow the reference."""
    g = golden("ref_random_n16")
    n = 16
    scene = W.make_scene(WL, PITCH, Z, n)
    pert = _perturbed(g["lut2"], 15, 17, 2.0 + 1.0j)
    lut = W.FringeLut(scene, 2, pert)
    assert not lut.support().flags.writeable  # value semantics: the device copy cannot go stale
    w = 1.25 + 0.5j
    ref, _ = O.ref_apply_block_lut(np.zeros((n, n)), pert, WL, PITCH, Z, 2, 4, 3, w)
    host = np.zeros((n, n), np.complex128)
    c = W.OpCounter()
    W.apply_block(host, lut, W.GridCell(4, 3), w, c, W.OpLevel.REFINE_FULL)
    assert O.max_rel_error(host, ref) <= 1e-6
    dev = W.DevicePlane(n)
    W.apply_block(dev, lut, W.GridCell(4, 3), w, c, W.OpLevel.REFINE_FULL)
    assert O.max_rel_error(dev.download(np.complex128), ref) <= 1e-6
    assert c.get(W.OpLevel.REFINE_FULL) == 2


@needs_ref
@pytest.mark.parametrize("name", ["ref_random_n16", "ref_random_n32"])
def test_progressive_from_stage_calls_on_a_device_plane(ctx, name):
    """synthesize_base + three refine calls (the stages of
    synthesis.cpp:216-251) with the reference's own LUT samples, accumulated
    in ONE device-resident plane (no host round trip between stages): every
    stage equals the reference's snapshot."""
    g = golden(name)
    n = g["object"].shape[0]
    scene = W.make_scene(WL, PITCH, Z, n)
    luts = W.LutSet()
    for b in (1, 2, 4, 8):
        luts.put(W.FringeLut(scene, b, g[f"lut{b}"]))
    pyr = W.haar_analyze(g["object"], 3)
    sal = W.quantize_saliency(g["saliency"])
    c = W.OpCounter()
    plane = W.DevicePlane(n).upload(W.synthesize_base(pyr, sal, luts, c))
    snaps = [plane.download(np.complex128)]
    for lvl, (factor, t, level) in enumerate(((4, 0.5, W.OpLevel.REFINE_LL),
                                              (2, 0.7, W.OpLevel.REFINE_L),
                                              (1, 0.9, W.OpLevel.REFINE_FULL))):
        det = pyr.details[2 - lvl]
        W.refine(plane, det.h, det.v, det.d, sal.by_factor(factor), luts.of(factor), t, c, level)
        snaps.append(plane.download(np.complex128))
    for s in range(4):
        assert O.rel_l2(snaps[s], g["planes"][s]) <= 1e-5, s
    assert [c.get(l) for l in W.OpLevel][:4] == g["ops"][:4].tolist()


@needs_ref
def test_lut_job_superposes_a_perturbed_caller_lutset_like_reference(ctx):
    """synthesize_progressive(..., luts) with one sample of the caller's B=1
    LUT changed: the LUT job (wcgh_job_use_lut) and the mirror move exactly
    like the reference's synthesize_progressive with the same LutSet."""
    g = golden("ref_random_n32")
    n = 32
    sups = {b: g[f"lut{b}"] for b in (1, 2, 4, 8)}
    pert = dict(sups)
    pert[1] = _perturbed(sups[1], n - 1, n - 1, 0.5 * np.abs(sups[1]).max() * (1 + 0.4j))
    pert[4] = _perturbed(sups[4], n + 2, n - 5, -0.5j * np.abs(sups[4]).max())
    ref0, ops0 = O.ref_synthesize_progressive_luts(g["object"], g["saliency"], WL, PITCH, Z, sups)
    ref1, ops1 = O.ref_synthesize_progressive_luts(g["object"], g["saliency"], WL, PITCH, Z, pert)
    assert np.allclose(ref0, g["planes"], rtol=0, atol=1e-12 * np.abs(g["planes"]).max())
    outs = []
    for s in (sups, pert):
        job = HologramJob(JobSpec(object_size=n, plane_size=n, layers=[(WL, PITCH, Z)],
                                  method="lut", obj_dtype="f64", sal_dtype="f64"))
        for b in (1, 2, 4, 8):
            job.use_lut(0, stages.DeviceLut((WL, PITCH, Z), n, b, s[b]))
        job(g["object"], g["saliency"])
        outs.append(job.download_stages().astype(np.complex128))
        assert job.stats()["ops"] == ops0.tolist()
        job.close()
    for st in range(4):
        assert O.rel_l2(outs[0][st], ref0[st]) <= 1e-5
        assert O.rel_l2(outs[1][st], ref1[st]) <= 1e-5
        d_ref, d_gpu = ref1[st] - ref0[st], outs[1][st] - outs[0][st]
        if st == 0:  # the base stage uses B = 8 only: untouched on both sides
            assert not d_ref.any() and not d_gpu.any()
            continue
        # both moved by the same field, up to the complex64 rounding of the
        # whole plane (the perturbation is well above that floor)
        floor = 3e-6 * np.linalg.norm(ref1[st])
        assert np.linalg.norm(d_ref) > 10 * floor, st
        assert np.linalg.norm(d_gpu - d_ref) <= floor, st
    # the Python mirror of synthesize_progressive with the same caller LutSet
    scene = W.make_scene(WL, PITCH, Z, n)
    luts = W.LutSet()
    for b in (1, 2, 4, 8):
        luts.put(W.FringeLut(scene, b, pert[b]))
    r = W.synthesize_progressive(g["object"], g["saliency"], scene, W.RefinementPlan(), luts)
    for st in range(4):
        assert O.rel_l2(r.stage(st), ref1[st]) <= 1e-5
    # a LUT for another scene is refused (synthesis.cpp:193-195)
    job = HologramJob(JobSpec(object_size=n, plane_size=n, layers=[(WL, PITCH, Z)], method="lut",
                              obj_dtype="f64", sal_dtype="f64"))
    with pytest.raises(_lib.ValidationError):
        job.use_lut(0, stages.DeviceLut((WL, PITCH, 0.2), n, 1, sups[1]))
    with pytest.raises(_lib.ValidationError):
        job.use_lut(0, stages.DeviceLut((WL, PITCH, Z), 16, 1, golden("ref_random_n16")["lut1"]))
    job.close()


def test_device_plane_upload_download_roundtrip(ctx):
    rng = np.random.default_rng(5)
    a = (rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))).astype(np.complex64)
    p = stages.DevicePlane(64).upload(a)
    assert np.array_equal(p.download(), a)
    assert np.array_equal(p.download(np.complex128), a.astype(np.complex128))
    p.zero()
    assert not p.download().any()
    with pytest.raises(_lib.ValidationError):
        p.upload(a[:32])
    bad = a.astype(np.complex128)
    bad[1, 1] = complex(np.inf, 0)
    with pytest.raises(_lib.ValidationError):
        p.upload(bad)
