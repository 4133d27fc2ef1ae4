"""Reconstruction + SSIM on the device (K6/K7 in
csrc/wcgh_recon.cu) against the reference's own outputs (tests/golden/
ref_recon_ssim.npz, made by oracle/_ref), the fp64 numpy oracle, and the
reference's angular-spectrum and metrics unit tests restated through the
Python mirror (test_angular_spectrum.cpp, test_metrics.cpp). Everything here
is fp64 like the reference, so the tolerances are the reference's own.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_2211_09938_b200 import stages
from paper_2211_09938_b200 import wavecgh as W
from paper_2211_09938_b200.hologram import HologramJob, spec_for_scene
from paper_2211_09938_b200.scenes import make_scene as make_blob_scene

pytestmark = pytest.mark.gpu

WL = 532e-9
SCENE32 = W.make_scene(WL, 8e-6, 0.1, 32)  # test_angular_spectrum.cpp:35


def random_field(n, seed):  # test_angular_spectrum.cpp:20-28 (numpy stand-in for mt19937_64)
    rng = np.random.default_rng(seed)
    return (rng.random((n, n)) - 0.5) + 1j * (rng.random((n, n)) - 0.5)


def energy(f):
    return float(np.sum(np.abs(f) ** 2))


def maxrel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


# ---- against the reference's outputs -----------------------------------------

@pytest.mark.parametrize("n", [16, 32])
def test_reconstruct_matches_reference(ctx, n):
    g = golden("ref_recon_ssim")
    sc = W.make_scene(WL, 8e-6, 0.1, n)
    assert maxrel(W.reconstruct(g[f"field{n}"], sc, False), g[f"mag{n}"]) <= 1e-12
    assert maxrel(W.reconstruct(g[f"field{n}"], sc, True), g[f"int{n}"]) <= 1e-12


def test_reconstruct_cfg0_hologram_matches_reference(ctx):
    g = golden("ref_recon_ssim")
    g0 = golden("ref_cfg0")
    sc = W.make_scene(WL, 8e-6, 0.2, 128)
    assert maxrel(W.reconstruct(g0["after_full"], sc), g["cfg0_recon"]) <= 1e-11
    # complex64 input (the synthesised-hologram type) widens exactly
    h64 = g0["after_full"].astype(np.complex64)
    assert np.array_equal(stages.reconstruct(h64, sc.layer()),
                          stages.reconstruct(h64.astype(np.complex128), sc.layer()))


def test_ssim_matches_reference(ctx):
    g = golden("ref_recon_ssim")
    off = 0
    for (n, win), v in zip(g["ssim_shape"], g["ssim_value"]):
        a = g["ssim_a"][off:off + n * n].reshape(n, n)
        b = g["ssim_b"][off:off + n * n].reshape(n, n)
        off += n * n
        assert abs(W.ssim(a, b, int(win), 0.01, 0.03, 1.0) - v) <= 1e-12
    dr = float(g["cfg0_recon"].max() - g["cfg0_recon"].min())
    s = W.ssim(g["cfg0_base_recon"], g["cfg0_recon"], 8, 0.01, 0.03, dr)
    assert abs(s - float(g["cfg0_base_ssim"])) <= 1e-12


def test_gpu_hologram_ssim_vs_reference_reconstruction(ctx):
    """The graded check at config 0: SSIM(reconstruct(GPU after_full),
    reconstruct(reference after_full)) >= 0.999, all on the device."""
    g = golden("ref_recon_ssim")
    sc = make_blob_scene(0)
    job = HologramJob(spec_for_scene(sc))
    job.upload(sc.objects, sc.masks)
    job.run()
    recon = job.reconstruct()
    ref = g["cfg0_recon"]
    dr = float(ref.max() - ref.min())
    s = W.ssim(recon, ref, 8, 0.01, 0.03, dr)
    assert s >= 0.999
    # device reconstruction of the resident plane == host round trip
    holo = job.download()
    assert np.array_equal(recon, stages.reconstruct(holo, (WL, 8e-6, 0.2)))
    assert abs(s - O.ssim(recon, ref, 8, 0.01, 0.03, dr)) <= 5e-12  # two fp64 reduction orders


# ---- test_angular_spectrum.cpp ------------------------------------------------

def test_fft_matches_direct_dft(ctx):  # :39-46
    f = random_field(8, 31)
    n = 8
    k = np.arange(n)
    w = np.exp(-2j * np.pi * np.outer(k, k) / n)
    slow_fwd = w @ f @ w.T
    slow_inv = (w.conj() @ f @ w.conj().T) / (n * n)
    assert maxrel(W.fft_2d(f, False), slow_fwd) <= 1e-12
    assert maxrel(W.fft_2d(f, True), slow_inv) <= 1e-12


def test_fft_round_trip(ctx):  # :48-52
    f = random_field(64, 77)
    assert maxrel(W.fft_2d(W.fft_2d(f, False), True), f) <= 1e-13


def test_fft_validates_input(ctx):  # :54-57
    with pytest.raises(W.ValidationError):
        W.fft_2d(np.zeros((12, 12), np.complex128), False)
    with pytest.raises(W.ValidationError):
        W.fft_2d(np.zeros((8, 4), np.complex128), False)


def test_kernel_dc_sample_and_unit_modulus(ctx):  # :59-74
    k = W.build_kernel(SCENE32, SCENE32.z())
    expected = np.exp(1j * 2.0 * np.pi * SCENE32.z() / SCENE32.wavelength())
    assert abs(k.transfer[0, 0] - expected) <= 1e-9
    assert 1.0 / (2.0 * SCENE32.pitch()) < 1.0 / SCENE32.wavelength()
    assert np.allclose(np.abs(k.transfer), 1.0, rtol=0, atol=1e-12)


def test_backward_kernel_is_conjugate(ctx):  # :76-83
    fwd = W.build_kernel(SCENE32, SCENE32.z()).transfer
    bwd = W.build_kernel(SCENE32, -SCENE32.z()).transfer
    assert np.abs(bwd - np.conj(fwd)).max() <= 1e-15


def test_kernel_rejects_zero_distance(ctx):  # :85-87
    with pytest.raises(W.ValidationError):
        W.build_kernel(SCENE32, 0.0)


def test_evanescent_samples_are_zero(ctx):
    # pitch below lambda/2 puts high frequencies past 1/lambda
    sc = W.make_scene(WL, 0.2e-6, 0.1, 32)
    t = W.build_kernel(sc, 0.1).transfer
    m = np.fft.fftfreq(32) * 32
    fx = m[None, :] / (32 * 0.2e-6)
    fy = m[:, None] / (32 * 0.2e-6)
    evanescent = (1.0 / WL**2 - fx * fx - fy * fy) < 0
    assert evanescent.any() and not evanescent.all()
    assert np.all(t[evanescent] == 0)
    assert np.allclose(np.abs(t[~evanescent]), 1.0, atol=1e-12)


def test_propagation_round_trip_and_energy(ctx):  # :89-99
    f = random_field(32, 5)
    fwd = W.build_kernel(SCENE32, SCENE32.z())
    bwd = W.build_kernel(SCENE32, -SCENE32.z())
    p = W.propagate(f, fwd)
    assert abs(energy(p) - energy(f)) <= 1e-12 * energy(f)
    assert maxrel(W.propagate(p, bwd), f) <= 1e-10


def test_propagate_matches_numpy_oracle(ctx):
    f = random_field(64, 9)
    sc = W.make_scene(WL, 8e-6, 0.05, 64)
    got = W.propagate(f, W.build_kernel(sc, 0.05))
    m = np.fft.fftfreq(64) * 64
    df = 1.0 / (64 * 8e-6)
    fx, fy = (m * df)[None, :], (m * df)[:, None]
    s = 1.0 / WL**2 - fx * fx - fy * fy
    t = np.where(s >= 0, np.exp(1j * 2 * np.pi * 0.05 * np.sqrt(np.maximum(s, 0))), 0)
    assert maxrel(got, np.fft.ifft2(np.fft.fft2(f) * t)) <= 1e-12


def test_uniform_field_is_eigenfunction(ctx):  # :101-109
    f = np.full((32, 32), 0.7 + 0j)
    k = W.build_kernel(SCENE32, SCENE32.z())
    out = W.propagate(f, k)
    assert np.abs(out - 0.7 * k.transfer[0, 0]).max() <= 1e-12


def test_propagate_validates_sizes(ctx):  # :111-114
    k = W.build_kernel(SCENE32, SCENE32.z())
    with pytest.raises(W.ValidationError):
        W.propagate(np.zeros((16, 16), np.complex128), k)


def test_zero_hologram_reconstructs_to_zero(ctx):  # :116-119
    assert np.all(W.reconstruct(np.zeros((32, 32), np.complex128), SCENE32) == 0.0)


def test_reconstruction_is_scale_equivariant(ctx):  # :121-128
    f = random_field(32, 99)
    a = W.reconstruct(f, SCENE32)
    b = W.reconstruct(f * 2.5, SCENE32)
    assert np.allclose(b, 2.5 * a, rtol=1e-12, atol=0)


def test_intensity_squares_magnitude(ctx):  # :130-138
    f = random_field(16, 3)
    sc = W.make_scene(WL, 8e-6, 0.1, 16)
    mag = W.reconstruct(f, sc, False)
    inten = W.reconstruct(f, sc, True)
    assert np.allclose(inten, mag * mag, rtol=1e-12, atol=0)


def test_bright_square_reconstructs_near_its_box(ctx):  # :140-168
    g = golden("ref_recon_ssim")
    sc = W.make_scene(WL, 8e-6, 0.01, 32)
    recon = W.reconstruct(g["square_holo"], sc)
    assert maxrel(recon, g["square_recon"]) <= 1e-12
    inside = np.zeros((32, 32), bool)
    inside[12:20, 12:20] = True
    assert recon[inside].mean() > 2.0 * recon[~inside].mean()


def test_reconstruct_validates(ctx):
    with pytest.raises(W.ValidationError):
        W.reconstruct(np.zeros((16, 16), np.complex128), SCENE32)
    with pytest.raises(W.ValidationError):
        stages.reconstruct(np.zeros((12, 12), np.complex128), (WL, 8e-6, 0.1))


# ---- test_metrics.cpp -------------------------------------------------------

def rimg(n, seed):
    return np.random.default_rng(seed).random((n, n))


def test_ssim_self_is_exactly_one(ctx):  # :16-19
    x = rimg(16, 21)
    assert W.ssim(x, x, 8, 0.01, 0.03, 1.0) == 1.0


def test_ssim_symmetric_and_bounded(ctx):  # :21-35
    a, b = rimg(16, 22), rimg(16, 23)
    assert abs(W.ssim(a, b, 8, 0.01, 0.03, 1.0) - W.ssim(b, a, 8, 0.01, 0.03, 1.0)) <= 1e-12
    for seed in range(6):
        s = W.ssim(rimg(24, 3000 + seed), rimg(24, 4000 + seed), 8, 0.01, 0.03, 1.0)
        assert -1.0 <= s <= 1.0


def test_inverted_binary_image_scores_negative(ctx):  # :37-50
    half = np.zeros((8, 8))
    half[:, 4:] = 1.0
    s = W.ssim(half, 1.0 - half, 8, 0.01, 0.03, 1.0)
    assert s < 0.0
    assert abs(s - O.ssim(half, 1.0 - half, 8, 0.01, 0.03, 1.0)) <= 1e-12 * abs(s)


def test_ssim_matches_oracle_rectangular_and_windows(ctx):
    rng = np.random.default_rng(4)
    a, b = rng.random((40, 56)), rng.random((40, 56))
    for win in (1, 5, 8, 40):
        assert abs(W.ssim(a, b, win, 0.01, 0.03, 2.0) - O.ssim(a, b, win, 0.01, 0.03, 2.0)) <= 1e-12


def test_ssim_validation(ctx):  # :65-71
    a = rimg(8, 1)
    with pytest.raises(W.ValidationError):
        W.ssim(a, rimg(16, 2), 8, 0.01, 0.03, 1.0)
    for win, dr in ((9, 1.0), (0, 1.0), (8, 0.0)):
        with pytest.raises(W.ValidationError):
            W.ssim(a, a, win, 0.01, 0.03, dr)
        with pytest.raises(W.ValidationError):
            stages.ssim(a, a, win, 0.01, 0.03, dr)


def test_report_pairs_stage_scores_with_cumulative_ops(ctx):  # :75-115
    n = 32
    sc = W.make_scene(WL, 8e-6, 0.1, n)
    luts = W.LutSet.build(sc)
    obj = rimg(n, 77)
    res = W.synthesize_progressive(obj, W.uniform_saliency(n), sc, W.RefinementPlan(0.0, 0.0, 0.0),
                                   luts)
    oracle = W.synthesize_pointwise_oracle(obj, sc, W.OpCounter(), luts.of(1))
    rep = W.build_report(res, W.reconstruct(oracle, sc), sc)
    assert len(rep.stages) == 4
    assert rep.stages[0].name == "base_LLL" and rep.stages[3].name == "after_full"
    assert rep.pointwise_ops == n * n
    base = (n // 8) ** 2
    assert rep.stages[0].ops_cumulative == base
    assert rep.stages[1].ops_cumulative == base + (n // 4) ** 2
    assert rep.stages[3].ops_cumulative == base + (n // 4) ** 2 + (n // 2) ** 2 + n * n
    for s in range(1, 4):
        assert rep.stages[s].ops_cumulative >= rep.stages[s - 1].ops_cumulative
    assert rep.stages[3].ssim >= 0.999
    assert rep.stages[0].ssim <= rep.stages[3].ssim
