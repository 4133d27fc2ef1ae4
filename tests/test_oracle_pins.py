"""Pins the fp64 C restatement (oracle/) against the reference: its golden
vectors (tests/golden/, produced by the reference itself) and, when it was
built here, the reference library (oracle/_ref). Restates the reference's
own known-answer tests."""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

WL = 532e-9


@pytest.mark.parametrize("name", ["ref_random_n16", "ref_random_n32"])
def test_oracle_matches_reference_goldens(name):
    g = golden(name)
    n = g["object"].shape[0]
    assert np.array_equal(O.haar_analyze(g["object"]), g["pyramid"])
    assert np.array_equal(O.quantize_saliency(g["saliency"]), g["sal_pyr"])
    luts = [O.build_block_lut(WL, 8e-6, 0.1, n, b) for b in (1, 2, 4, 8)]
    for b, lut in zip((1, 2, 4, 8), luts):
        assert np.abs(lut - g[f"lut{b}"]).max() <= 1e-12 * np.abs(g[f"lut{b}"]).max()
    planes, masks, ops = O.synthesize_progressive(g["object"], g["saliency"], WL, 8e-6, 0.1,
                                                  luts=luts)
    assert np.array_equal(masks, g["masks"]) and np.array_equal(ops, g["ops"])
    for s in range(4):
        assert O.max_rel_error(planes[s], g["planes"][s]) <= 1e-12


def test_a_eff_identity_pins_the_direct_oracle():
    # after_full == pointwise_sum(A_eff) (SURVEY.md §0 finding 1), on the
    # reference's own cfg0 output
    g = golden("ref_cfg0")
    an = O.analysis(g["object"].astype(np.float64), g["mask"] * (1.0 / 255.0))
    assert np.array_equal(an["masks"], g["masks"]) and np.array_equal(an["ops"], g["ops"])
    assert np.array_equal(an["pyramid"], g["pyramid"])
    xs, ys, amps, lay = O.compact(an["a_eff"])
    n = 128
    rows = np.arange(0, n, 9)  # a pixel subset keeps this CPU test fast
    py, px = np.meshgrid(rows, np.arange(n), indexing="ij")
    h = O.direct_pixels(xs, ys, amps, lay, [(WL, 8e-6, 0.2)], px.ravel(), py.ravel())
    ref = g["after_full"][py.ravel(), px.ravel()]
    assert O.max_rel_error(h, ref) <= 1e-9


def test_padded_and_layered_conventions():
    g = golden("ref_padded_32on64")
    xs, ys, amps, lay, ops = O.scene_points(g["object"][None].astype(np.float64),
                                            g["mask"][None] * (1.0 / 255.0), 64)
    yy, xx = np.mgrid[0:64, 0:64]
    h = O.direct_pixels(xs, ys, amps, lay, [(WL, 8e-6, 0.05)], xx.ravel(), yy.ravel())
    assert O.max_rel_error(h.reshape(64, 64), g["after_full"]) <= 1e-9
    g = golden("ref_two_layers_64")
    xs, ys, amps, lay, ops = O.scene_points(g["objects"], g["saliency"], 64)
    h = O.direct_pixels(xs, ys, amps, lay, [(WL, 8e-6, z) for z in g["depths"]], xx.ravel(),
                        yy.ravel())
    assert O.max_rel_error(h.reshape(64, 64), g["after_full"]) <= 1e-9


def test_telescoping_and_opcounts():
    g = golden("ref_telescoping_n32")
    assert O.max_rel_error(g["after_full"], g["direct"]) <= 1e-9  # test_synthesis.cpp:193-203
    an = O.analysis(g["object"], np.ones((32, 32)), t=(0.0, 0.0, 0.0))
    assert np.abs(an["a_eff"] - g["object"]).max() <= 1e-14  # full refinement: A_eff == object
    # acceptance_main.cpp:92-122 at 256^2: 1024 / 5120 / 21504 / 87040 cumulative
    assert np.cumsum(golden("ref_opcounts_256")["ops"][:4]).tolist() == [1024, 5120, 21504, 87040]
    an = O.analysis(np.random.default_rng(0).random((256, 256)), np.ones((256, 256)), t=(0, 0, 0))
    assert np.cumsum(an["ops"][:4]).tolist() == [1024, 5120, 21504, 87040]


def test_known_answers():
    # test_haar.cpp:38-53 impulse, 88-97 residual sign pattern
    img = np.zeros((2, 2))
    img[0, 0] = 1.0
    assert O.haar_analyze(img, 1).tolist() == [0.25, 0.25, 0.25, 0.25]
    r = O.expand_residual(np.array([[0.25]]), np.array([[0.25]]), np.array([[0.25]]))
    assert r.tolist() == [[0.75, -0.25], [-0.25, -0.25]]
    # test_fringe_lut.cpp:26-31 on-axis |F| = 1/z
    out = np.empty(2)
    O.orc().orc_point_fringe(WL, 8e-6, 0.1, 0, 0, out.ctypes.data)
    assert abs(np.hypot(*out) - 10.0) <= 1e-13
    g = golden("ref_point_fringe")
    for (dx, dy), val in zip(g["offsets"], g["values"]):
        O.orc().orc_point_fringe(WL, 8e-6, 0.1, int(dx), int(dy), out.ctypes.data)
        assert abs(complex(*out) - val) <= 1e-12 * abs(val)
    # test_saliency.cpp: a single salient pixel propagates to every level
    m = np.zeros((16, 16))
    m[0, 0] = 1.0
    sp = O.quantize_saliency(m)
    assert sp.sum() == 3.0 and sp[0] == 1.0
    with pytest.raises(ValueError):
        O.quantize_saliency(np.full((8, 8), 1.5))


def test_lut_composition():
    # test_fringe_lut.cpp:92-112 / acceptance 6: a B-LUT is the sum of four B/2 LUTs
    n = 16
    for b in (2, 4, 8):
        parent = O.build_block_lut(WL, 8e-6, 0.1, n, b)
        child = O.build_block_lut(WL, 8e-6, 0.1, n, b // 2)
        h = b // 2
        o = n - 1
        worst = 0.0
        for dy in range(-(n - 1) + h, n):
            for dx in range(-(n - 1) + h, n):
                s = (child[dy + o, dx + o] + child[dy + o, dx - h + o] + child[dy - h + o, dx + o]
                     + child[dy - h + o, dx - h + o])
                worst = max(worst, abs(parent[dy + o, dx + o] - s))
        assert worst <= 1e-12 * np.abs(parent).max()


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_matches_reference_library_live():
    rng = np.random.default_rng(7)
    for n in (8, 16, 64):
        obj = rng.integers(0, 256, (n, n)).astype(np.float64)
        sal = rng.random((n, n))
        assert np.array_equal(O.haar_analyze(obj), O.ref_haar_analyze(obj))
        p1, m1, o1 = O.synthesize_progressive(obj, sal, WL, 8e-6, 0.1)
        p2, m2, o2 = O.ref_synthesize_progressive(obj, sal, WL, 8e-6, 0.1)
        assert np.array_equal(m1, m2) and np.array_equal(o1, o2)
        assert O.max_rel_error(p1[3], p2[3]) <= 1e-12
    h = golden("ref_cfg0")["after_full"]
    r1 = O.reconstruct(h, WL, 8e-6, 0.2)
    r2 = O.ref_reconstruct(h, WL, 8e-6, 0.2)
    assert np.abs(r1 - r2).max() <= 1e-12 * np.abs(r2).max()
    dr = r2.max() - r2.min()
    assert abs(O.ssim(r1, r2 * 0.97, 8, 0.01, 0.03, dr) - O.ref_ssim(r1, r2 * 0.97, 8, 0.01, 0.03, dr)) < 1e-12


def test_fft_oracle_matches_reference_and_direct_sum():
    # the full-plane fp64 FFT oracle reproduces the reference's own outputs...
    g = golden("ref_cfg0")
    an = O.analysis(g["object"].astype(np.float64), g["mask"] * (1.0 / 255.0))
    h = O.fft_hologram(an["a_eff"], [(WL, 8e-6, 0.2)], 128)
    assert O.max_rel_error(h, g["after_full"]) <= 1e-10
    g = golden("ref_padded_32on64")
    a = O.analysis(g["object"].astype(np.float64), g["mask"] * (1.0 / 255.0))["a_eff"]
    assert O.max_rel_error(O.fft_hologram(a, [(WL, 8e-6, 0.05)], 64), g["after_full"]) <= 1e-10
    g = golden("ref_two_layers_64")
    a = O.scene_a_eff(g["objects"], g["saliency"])
    h = O.fft_hologram(a, [(WL, 8e-6, z) for z in g["depths"]], 64)
    assert O.max_rel_error(h, g["after_full"]) <= 1e-10
    # ...and the direct Eq.(1) oracle on an object smaller than the plane
    from paper_2211_09938_b200 import scenes

    sc = scenes.make_scene(scenes.SceneConfig("t", 0, 64, 256, 8e-6, (0.2,)))
    a = O.scene_a_eff(sc.objects.astype(np.float64), sc.masks / 255.0)
    h = O.fft_hologram(a, [(WL, 8e-6, 0.2)], 256)
    xs, ys, amps, lay = O.compact(a[0], off=96)
    rng = np.random.default_rng(2)
    px, py = rng.integers(0, 256, 300), rng.integers(0, 256, 300)
    ref = O.direct_pixels(xs, ys, amps, lay, [(WL, 8e-6, 0.2)], px, py)
    assert O.max_rel_error(h[py, px], ref) <= 1e-10


def test_recon_and_ssim_oracles_match_reference_goldens():
    """oracle.reconstruct (numpy fp64 FFT) and oracle.ssim (C restatement of
    metrics.cpp:49-85) against the reference's own outputs."""
    g = golden("ref_recon_ssim")
    for n in (16, 32):
        for key, inten in (("mag", False), ("int", True)):
            r = O.reconstruct(g[f"field{n}"], WL, 8e-6, 0.1, intensity=inten)
            ref = g[f"{key}{n}"]
            assert np.abs(r - ref).max() <= 1e-12 * np.abs(ref).max()
    g0 = golden("ref_cfg0")
    r = O.reconstruct(g0["after_full"], WL, 8e-6, 0.2)
    assert np.abs(r - g["cfg0_recon"]).max() <= 1e-11 * g["cfg0_recon"].max()
    off = 0
    for (n, win), v in zip(g["ssim_shape"], g["ssim_value"]):
        a = g["ssim_a"][off:off + n * n].reshape(n, n)
        b = g["ssim_b"][off:off + n * n].reshape(n, n)
        off += n * n
        assert abs(O.ssim(a, b, int(win)) - v) <= 1e-12


def test_random_phase_field_and_complex_restatement_pins():
    """random_phase_field (synthesis.cpp:288-296) through the library's host
    function — the reference's own engine, no device work — is bit-identical
    to the reference's; the complex synthesis restated by linearity (pyr_re,
    pyr_im; synthesis.cpp:205-251) reproduces the reference's snapshots."""
    from paper_2211_09938_b200 import stages
    g = golden("ref_random_phase")
    for n in (16, 32):
        obj, sal, rot = g[f"object{n}"], g[f"saliency{n}"], g[f"rotated{n}"]
        assert np.array_equal(stages.random_phase_field(obj, int(g[f"seed{n}"])), rot)
        assert np.allclose(np.abs(rot), obj, rtol=1e-12, atol=0)  # test_synthesis.cpp:425-431
        luts = [O.build_block_lut(WL, 8e-6, 0.1, n, b) for b in (1, 2, 4, 8)]
        pr, masks, ops = O.synthesize_progressive(rot.real, sal, WL, 8e-6, 0.1, luts=luts)
        pi, masks_i, _ = O.synthesize_progressive(rot.imag, sal, WL, 8e-6, 0.1, luts=luts)
        assert np.array_equal(masks, g[f"masks{n}"]) and np.array_equal(masks_i, masks)
        assert np.array_equal(ops, g[f"ops{n}"])
        for s in range(4):
            assert O.max_rel_error(pr[s] + 1j * pi[s], g[f"planes{n}"][s]) <= 1e-12
        # telescoping: == the direct sum of the rotated field
        assert O.max_rel_error(g[f"tele{n}"], g[f"direct{n}"]) <= 1e-9
