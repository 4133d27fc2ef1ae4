"""Generates tests/golden/*.npz from the REFERENCE ITSELF.

Runs the unmodified reference sources (oracle/_ref/libwavecgh_ref.so, built
by oracle/Makefile from /root/reference/proj) on seeded inputs and stores
inputs + outputs as small fixtures. /root/reference does not exist on the GPU
box, so the GPU tests and the CPU oracle pins read these files instead.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2211_09938_b200 import scenes  # noqa: E402

OUT = Path(__file__).resolve().parent
WL = 532e-9


def save(name: str, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(name, {k: (v.shape, v.dtype) for k, v in arrays.items()})


def main():
    assert O.ref_available(), "oracle/_ref not built (needs /root/reference)"

    # 1. Reference unit-test geometry (test_synthesis.cpp:17): z = 0.1, pitch 8 um;
    #    random_image (mt19937_64) objects and saliency, default plan.
    for n, seed in ((16, 8), (32, 5)):
        obj = O.ref_random_image(n, n, seed)
        sal = O.ref_random_image(n, n, seed + 1)
        pyr = O.ref_haar_analyze(obj, 3)
        sp = O.ref_quantize_saliency(sal)
        planes, masks, ops = O.ref_synthesize_progressive(obj, sal, WL, 8e-6, 0.1)
        luts = {f"lut{b}": O.ref_build_block_lut(WL, 8e-6, 0.1, n, b) for b in (1, 2, 4, 8)}
        save(f"ref_random_n{n}", object=obj, saliency=sal, pyramid=pyr, sal_pyr=sp,
             planes=planes, masks=masks, ops=ops, **luts)

    # 2. Telescoping: uniform saliency, zero thresholds (test_synthesis.cpp:193-203).
    n = 32
    obj = O.ref_random_image(n, n, 900 + n)
    planes, masks, ops = O.ref_synthesize_progressive(obj, np.ones((n, n)), WL, 8e-6, 0.1,
                                                      t=(0.0, 0.0, 0.0))
    direct = O.ref_pointwise_hologram_reference(obj, WL, 8e-6, 0.1)
    save("ref_telescoping_n32", object=obj, after_full=planes[3], direct=direct, ops=ops)

    # 3. Config 0 (BASELINE.json configs[0]): 128^2 blob object (uint8 values
    #    as amplitudes), 25% mask, z = 0.2, pitch 8 um, default plan.
    sc = scenes.make_scene(0)
    obj = sc.objects[0].astype(np.float64)
    sal = sc.masks[0].astype(np.float64) * (1.0 / 255.0)
    planes, masks, ops = O.ref_synthesize_progressive(obj, sal, WL, 8e-6, 0.2)
    save("ref_cfg0", object=sc.objects[0], mask=sc.masks[0], after_full=planes[3],
         base=planes[0], masks=masks, ops=ops, pyramid=O.ref_haar_analyze(obj, 3))

    # 4. Centring convention for No < Nh: the reference run on the object
    #    zero-padded to the centre of a 64^2 plane.
    sc = scenes.make_scene(scenes.SceneConfig("pad", 0, 32, 64, 8e-6, (0.05,)))
    No, Nh = 32, 64
    off = (Nh - No) // 2
    objp = np.zeros((Nh, Nh))
    salp = np.zeros((Nh, Nh))
    objp[off:off + No, off:off + No] = sc.objects[0]
    salp[off:off + No, off:off + No] = sc.masks[0] * (1.0 / 255.0)
    planes, masks, ops = O.ref_synthesize_progressive(objp, salp, WL, 8e-6, 0.05)
    save("ref_padded_32on64", object=sc.objects[0], mask=sc.masks[0], after_full=planes[3],
         ops=ops)

    # 5. Two depth layers on a 64^2 plane: the per-layer reference sum.
    objs, sals, total = [], [], np.zeros((64, 64), np.complex128)
    for layer, z in enumerate((0.05, 0.08)):
        o = (O.ref_random_image(64, 64, 70 + layer) * 255).round()
        s = (O.ref_random_image(64, 64, 80 + layer) > 0.6).astype(np.float64)
        planes, masks, ops = O.ref_synthesize_progressive(o, s, WL, 8e-6, z)
        objs.append(o), sals.append(s)
        total += planes[3]
    save("ref_two_layers_64", objects=np.stack(objs), saliency=np.stack(sals), after_full=total,
         depths=np.array([0.05, 0.08]))

    # 6. Acceptance 2 (acceptance_main.cpp:92-122): op counts at 256^2.
    n = 256
    obj = O.ref_random_image(n, n, 7)
    _, _, ops = O.ref_synthesize_progressive(obj, np.ones((n, n)), WL, 8e-6, 0.1,
                                             t=(0.0, 0.0, 0.0))
    save("ref_opcounts_256", ops=ops)

    # 7. point_fringe samples (fringe_lut.cpp:27-32) incl. the long-double
    #    case of test_fringe_lut.cpp:41-58.
    pts = [(0, 0), (5, -3), (-5, 3), (3, 5), (100, 0), (1000, 700), (-2559, 3071)]
    vals = np.array([O.ref_point_fringe(WL, 8e-6, 0.1, 256, dx, dy) for dx, dy in pts])
    save("ref_point_fringe", offsets=np.array(pts, np.int32), values=vals)

    # 8. Reconstruction + SSIM (angular_spectrum.cpp:47-61, metrics.cpp:49-85):
    #    random complex fields as in test_angular_spectrum.cpp:20-28, the
    #    config-0 reference hologram, the bright-square hologram of
    #    test_angular_spectrum.cpp:140-150, and SSIM pairs of test_metrics.cpp.
    rec = {}
    for n, seed in ((16, 3), (32, 99)):
        f = (O.ref_random_image(n, n, seed) - 0.5) + 1j * (O.ref_random_image(n, n, seed + 1) - 0.5)
        rec[f"field{n}"] = f
        rec[f"mag{n}"] = O.ref_reconstruct(f, WL, 8e-6, 0.1, False)
        rec[f"int{n}"] = O.ref_reconstruct(f, WL, 8e-6, 0.1, True)
    g0 = np.load(OUT / "ref_cfg0.npz")
    rec["cfg0_recon"] = O.ref_reconstruct(g0["after_full"], WL, 8e-6, 0.2, False)
    rec["cfg0_base_recon"] = O.ref_reconstruct(g0["base"], WL, 8e-6, 0.2, False)
    dr = float(rec["cfg0_recon"].max() - rec["cfg0_recon"].min())
    rec["cfg0_base_ssim"] = np.array(O.ref_ssim(rec["cfg0_base_recon"], rec["cfg0_recon"], 8, 0.01,
                                                0.03, dr))
    sq = np.zeros((32, 32))
    sq[12:20, 12:20] = 1.0
    rec["square_holo"] = O.ref_pointwise_hologram_reference(sq, WL, 8e-6, 0.01)
    rec["square_recon"] = O.ref_reconstruct(rec["square_holo"], WL, 8e-6, 0.01, False)
    pairs = [(16, 5000, 6000, 8), (16, 5001, 6001, 8), (8, 7000, 7001, 8), (24, 3000, 4000, 3),
             (24, 3001, 4001, 16), (32, 11, 12, 1)]
    sa, sb, sw, sv = [], [], [], []
    for n, s1, s2, win in pairs:
        a = O.ref_random_image(n, n, s1)
        b = O.ref_random_image(n, n, s2)
        sa.append(a.ravel()), sb.append(b.ravel()), sw.append((n, win))
        sv.append(O.ref_ssim(a, b, win, 0.01, 0.03, 1.0))
    rec["ssim_a"] = np.concatenate(sa)
    rec["ssim_b"] = np.concatenate(sb)
    rec["ssim_shape"] = np.array(sw, np.int32)
    rec["ssim_value"] = np.array(sv)
    save("ref_recon_ssim", **rec)

    # 9. A CGHL LUT cache file written by the reference (lut_cache_store,
    #    fringe_lut.cpp:95-115): 16^2 plane, block 2, z = 0.1.
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        path = Path(td) / "lut.cghl"
        O.ref_lut_cache_store(path, WL, 8e-6, 0.1, 16, 2)
        save("ref_cghl_n16_b2", cghl_bytes=np.frombuffer(path.read_bytes(), np.uint8),
             lut=O.ref_build_block_lut(WL, 8e-6, 0.1, 16, 2))
    random_phase()


def random_phase():
    """10. Random initial phase (synthesis.cpp:205-219, 269-296): the rotated
    object, the four snapshots under the default plan, the telescoping case of
    test_synthesis.cpp:408-433 (uniform saliency, zero thresholds, vs the
    direct Eq.(1) sum of the rotated field) and the point-wise oracle."""
    out = {}
    for n, seed in ((16, 424242), (32, 77)):
        obj = O.ref_random_image(n, n, 13 + n)
        sal = O.ref_random_image(n, n, 14 + n)
        rot = O.ref_random_phase_field(obj, seed)
        planes, masks, ops = O.ref_synthesize_progressive(obj, sal, WL, 8e-6, 0.1, seed=seed)
        tele, _, tops = O.ref_synthesize_progressive(obj, np.ones((n, n)), WL, 8e-6, 0.1,
                                                     t=(0.0, 0.0, 0.0), seed=seed)
        pw, pops = O.ref_pointwise_oracle(obj, WL, 8e-6, 0.1, seed=seed)
        out.update({f"object{n}": obj, f"saliency{n}": sal, f"seed{n}": np.array(seed, np.uint64),
                    f"rotated{n}": rot, f"planes{n}": planes, f"masks{n}": masks, f"ops{n}": ops,
                    f"tele{n}": tele[3], f"tele_ops{n}": tops,
                    f"direct{n}": O.ref_pointwise_hologram_reference(rot, WL, 8e-6, 0.1),
                    f"pointwise{n}": pw, f"pointwise_ops{n}": np.array(pops, np.uint64)})
    save("ref_random_phase", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["--random-phase"]:
        random_phase()
    else:
        main()
