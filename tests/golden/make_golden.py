"""Generates the golden vectors in this directory from the REFERENCE ITSELF.

Run in a container that has /root/reference (the reference headers compiled behind
oracle/ref_shim.cpp by `make -C oracle ref`):

    python tests/golden/make_golden.py

The vectors pin the C restatement (oracle/ffdp_oracle.c) through
tests/test_oracle_golden.py, which runs anywhere (no /root/reference needed). Inputs
are regenerated from seeds with the reference's own splitmix64 Rng (rng.hpp), mirroring
the fixture patterns of the reference tests (test_sampler.cpp:30-61 margin fixture,
test_lncc.cpp, test_mi.cpp:56-69, test_distops.cpp).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import Oracle, Reference, step_inputs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def margin_fixture(orc, seed, img_shape, out_shape, perturb):
    """test_sampler.cpp:30-61: fractional source indices in [0.15, 0.85]."""
    r = orc.rng(seed)
    L = orc.lib
    import ctypes as C
    img = orc.random_volume(r, img_shape)
    S = np.array([1.25, 0.8, 1.1])
    A = np.eye(3)
    t = np.zeros(3)
    if perturb:
        for i in range(3):
            for j in range(3):
                A[i, j] = (1.0 if i == j else 0.0) + (-0.05 + 0.1 * L.or_rng_uniform(C.byref(r)))
        t = np.array([-0.05 + 0.1 * L.or_rng_uniform(C.byref(r)) for _ in range(3)])
    onz, ony, onx = out_shape
    inz, iny, inx = img_shape
    n_img = (inx, iny, inz)
    u = np.zeros(tuple(out_shape) + (3,))
    ax = lambda i, n: -1.0 + 2.0 * (i / (n - 1))
    for z in range(onz):
        for y in range(ony):
            for x in range(onx):
                X = np.array([ax(x, onx), ax(y, ony), ax(z, onz)])
                base = A @ X + t
                for c in range(3):
                    n = n_img[c]
                    cell = L.or_rng_uniform_int(C.byref(r), -1, n - 1)
                    frac = 0.15 + 0.7 * L.or_rng_uniform(C.byref(r))
                    target = 2.0 * (cell + frac) / (n - 1) - 1.0
                    u[z, y, x, c] = (target - base[c]) / S[c]
    return img, u, A, t, S


def label_maps(c1, c2, shape=(14, 16, 18)):
    """Two ellipsoids and a slab of labels 1-3 on a (nz, ny, nx) lattice."""
    nz, ny, nx = shape
    z, y, x = np.mgrid[:nz, :ny, :nx]
    a = np.zeros(shape, np.uint16)
    a[((x - c1[0]) ** 2 / 16 + (y - c1[1]) ** 2 / 9 + (z - c1[2]) ** 2 / 9) < 1] = 1
    a[((x - c2[0]) ** 2 / 6 + (y - c2[1]) ** 2 / 4 + (z - c2[2]) ** 2 / 5) < 1] = 2
    a[(x < 3) & (y > 10)] = 3
    return a


def nifti_fixtures(orc):
    """Files in tests/golden/nifti/ written by the reference's write_nifti / write_warp, two
    hand-made variants (big-endian, int16 with scl_slope), and the reference's parse of
    each (read_nifti / read_warp)."""
    import ctypes as C
    import struct
    so = os.path.join(ROOT, "oracle", "_ref", "libvoxreg_io.so")
    if not os.path.exists(so):
        raise SystemExit("make -C oracle ref-io first")
    L = C.CDLL(so)
    dp, i64p = C.POINTER(C.c_double), C.POINTER(C.c_int64)
    P = lambda a: a.ctypes.data_as(dp)
    d3 = lambda shape: (C.c_int64 * 3)(shape[2], shape[1], shape[0])
    nd = os.path.join(OUT, "nifti")
    os.makedirs(nd, exist_ok=True)
    g = {}
    v = orc.random_volume(orc.rng(951), (3, 5, 7), -2.0, 3.0)
    sp, og = np.array([0.7, 1.1, 2.5]), np.array([-10.0, 4.5, 0.25])
    for f64 in (0, 1):
        fn = os.path.join(nd, f"vol_f{64 if f64 else 32}.nii")
        assert L.refio_write_nifti(P(v), d3(v.shape), P(sp), P(og), f64, fn.encode()) == 0
    lab = (orc.random_volume(orc.rng(952), (4, 3, 6), 0, 300)).astype(np.uint16)
    assert L.refio_write_labels(lab.ctypes.data_as(C.POINTER(C.c_uint16)), d3(lab.shape), P(sp),
                                os.path.join(nd, "labels.nii").encode()) == 0
    # big-endian copy of the fp32 file: every header field and voxel byte-swapped
    b = bytearray(open(os.path.join(nd, "vol_f32.nii"), "rb").read())
    be = bytearray(b)
    struct.pack_into(">i", be, 0, 348)
    struct.pack_into(">8h", be, 40, *struct.unpack_from("<8h", b, 40))
    struct.pack_into(">2h", be, 70, *struct.unpack_from("<2h", b, 70))
    struct.pack_into(">8f", be, 76, *struct.unpack_from("<8f", b, 76))
    struct.pack_into(">3f", be, 108, *struct.unpack_from("<3f", b, 108))
    struct.pack_into(">3f", be, 268, *struct.unpack_from("<3f", b, 268))
    n = v.size
    be[352:] = np.frombuffer(bytes(b[352:352 + 4 * n]), dtype="<f4").astype(">f4").tobytes()
    open(os.path.join(nd, "vol_be.nii"), "wb").write(bytes(be))
    # int16 payload with scl_slope / scl_inter (a scanner-style file)
    sc = bytearray(open(os.path.join(nd, "labels.nii"), "rb").read())
    struct.pack_into("<2f", sc, 112, 0.5, -3.0)
    open(os.path.join(nd, "scaled_i16.nii"), "wb").write(bytes(sc))
    for name in ("vol_f32", "vol_f64", "labels", "vol_be", "scaled_i16"):
        fn = os.path.join(nd, name + ".nii").encode()
        dims, spo, ogo = (C.c_int64 * 3)(), np.zeros(3), np.zeros(3)
        assert L.refio_read_nifti(fn, dims, P(spo), P(ogo), None) == 0
        out = np.zeros((dims[2], dims[1], dims[0]))
        assert L.refio_read_nifti(fn, dims, P(spo), P(ogo), P(out)) == 0
        g.update({f"nii_{name}": out, f"nii_{name}_spacing": spo, f"nii_{name}_origin": ogo})
    g.update({"nii_src": v, "nii_src_spacing": sp, "nii_src_origin": og, "nii_labels_src": lab.astype(np.int64)})
    w = orc.random_volume(orc.rng(953), (3, 4, 5, 3), -0.1, 0.1)
    assert L.refio_write_warp(P(w), d3(w.shape[:3]), P(sp), P(og), os.path.join(nd, "warp").encode()) == 0
    dims = (C.c_int64 * 3)()
    wo = np.zeros_like(w)
    assert L.refio_read_warp(os.path.join(nd, "warp").encode(), dims, P(wo)) == 0
    g.update({"warp_src": w, "warp_read": wo})
    return g


def main():
    orc, ref = Oracle(), Reference()
    g = {}
    # --- sampler: margin fixtures (fwd + every gradient), distinct in/out lattices
    for i, (ish, osh, pert) in enumerate([((8, 8, 8), (8, 8, 8), True), ((7, 7, 7), (6, 6, 6), True),
                                          ((6, 9, 5), (5, 4, 7), False)]):
        img, u, A, t, S = margin_fixture(orc, 107 + i, ish, osh, pert)
        up = orc.random_volume(orc.rng(500 + i), osh, -1.0, 1.0)
        fw = ref.sample(img, u, A, t, S)
        bw = ref.sample(img, u, A, t, S, upstream=up, want=("image", "warp", "affine", "translation"))
        g.update({f"smp{i}_img": img, f"smp{i}_u": u, f"smp{i}_A": A, f"smp{i}_t": t, f"smp{i}_S": S,
                  f"smp{i}_up": up, f"smp{i}_out": fw["out"], f"smp{i}_gimg": bw["image"],
                  f"smp{i}_gu": bw["warp"], f"smp{i}_gA": bw["affine"], f"smp{i}_gt": bw["translation"]})
    # sampler on a face (test_sampler.cpp:225-241) and with sharded output bounds
    r = orc.rng(137)
    img = orc.random_volume(r, (6, 6, 6))
    u = np.zeros((6, 6, 6, 3))
    u[2, 2, 2, 0] = (2.0 * 3.0 / 5.0 - 1.0) - (-1.0 + 2.0 * 2 / 5)
    up = np.zeros((6, 6, 6))
    up[2, 2, 2] = 1.0
    bw = ref.sample(img, u, upstream=up, want=("warp",))
    g.update({"face_img": img, "face_u": u, "face_up": up, "face_gu": bw["warp"]})
    bounds = np.array([-1, -1, -0.2, 1, 1, 0.6])
    img = orc.random_volume(orc.rng(141), (9, 8, 7))
    u = orc.random_volume(orc.rng(142), (4, 8, 7, 3), -0.05, 0.05)
    fw = ref.sample(img, u, bounds=bounds)
    g.update({"bnd_img": img, "bnd_u": u, "bnd_bounds": bounds, "bnd_out": fw["out"]})

    # --- LNCC: fwd (loss, state, map) + bwd ANTs / exact, odd lattice, windows 7 and 3
    for i, (sh, w) in enumerate([((12, 11, 10), 7), ((9, 10, 13), 3), ((5, 6, 7), 7)]):
        r = orc.rng(211 + i)
        f = orc.random_volume(r, sh)
        m = orc.random_volume(r, sh)
        for ants in (True, False):
            res = ref.lncc(f, m, window=w, eps=1e-5, ants=ants, upstream=1.3, want_map=True)
            k = f"lncc{i}_{'ants' if ants else 'exact'}"
            g.update({f"{k}_loss": np.array(res["loss"]), f"{k}_gf": res["grad_f"], f"{k}_gm": res["grad_m"]})
        g.update({f"lncc{i}_f": f, f"lncc{i}_m": m, f"lncc{i}_w": np.array(w), f"lncc{i}_state": res["state"],
                  f"lncc{i}_map": res["map"]})

    # --- MI: exact / approx, three kernels, B = 8 and 32, margin-filled intensities
    r = orc.rng(311)
    vi = orc.random_volume(r, (6, 7, 8), 0.0, 1.0)
    vj = np.clip(0.6 * vi + 0.4 * orc.random_volume(r, (6, 7, 8)), 0, 1)
    g.update({"mi_i": vi, "mi_j": vj})
    for kind in ("gaussian", "bspline3", "delta"):
        for bins in (8, 32):
            for approx in (False, True):
                res = ref.mi(vi, vj, bins=bins, kind=kind, approx=approx, upstream=-1.0)
                k = f"mi_{kind}_{bins}_{int(approx)}"
                g.update({f"{k}_mi": np.array(res["mi"]), f"{k}_raw": res["raw"], f"{k}_pij": res["pij"],
                          f"{k}_stats": np.array(res["stats"], dtype=np.uint64), f"{k}_gi": res["grad_i"],
                          f"{k}_gj": res["grad_j"]})
    xs = np.linspace(-0.2, 0.2, 401)
    for kind in ("gaussian", "bspline3", "delta"):
        kap, om = ref.parzen_eval(kind, 32, xs)
        g.update({f"parzen_{kind}_kappa": kap, f"parzen_{kind}_omega": om})
    g["parzen_x"] = xs

    # --- synth pair + the full step at H = 1 and H = 2 / 3 (ring + halo + allreduce)
    f, m, w = ref.synth_pair(4242, (16, 17, 18), 5, 0.12)
    g.update({"synth_f": f, "synth_m": m, "synth_w": w})
    lf, lm, pre = ref.synth_labels(4242, (16, 17, 18), 5, 0.12)
    g.update({"synth_lf": lf, "synth_lm": lm, "synth_pre": pre})
    for loss in ("lncc", "mi"):
        si = step_inputs(orc, (18, 17, 16), seed=4242, loss=loss)
        g.update({f"step_{loss}_f": si.f, f"step_{loss}_m": si.m, f"step_{loss}_u": si.u, f"step_{loss}_A": si.A,
                  f"step_{loss}_t": si.t})
        for world in (1, 2, 3):
            res = ref.step(loss, si.f, si.m, si.u, si.A, si.t, world=world)
            g.update({f"step_{loss}_H{world}_loss": np.array(res["loss"]), f"step_{loss}_H{world}_gu": res["g_u"],
                      f"step_{loss}_H{world}_moved": res["moved"]})

    # --- gp_convolve across shards (distops.hpp:54-101)
    v = orc.random_volume(orc.rng(601), (11, 6, 5))
    for world in (1, 2, 3):
        for sync in (True, False):
            g[f"gp_box_H{world}_s{int(sync)}"] = ref.gp_convolve(v, np.full(7, 1 / 7), world, False, sync)
    g["gp_v"] = v
    wv = orc.random_volume(orc.rng(602), (9, 5, 4, 3))
    g["gp_w"] = wv
    g["gp_gauss_H3"] = ref.gp_convolve(wv, orc.gaussian_taps(1.0), 3, True, True)

    # --- the warp update (registration.hpp:313-317): gp_convolve(g_u) -> adam_step ->
    #     gp_convolve(u), two consecutive Adam steps, H = 1 and 3
    r = orc.rng(701)
    sh = (11, 9, 10)
    wu_g = orc.random_volume(r, sh + (3,), -1e-3, 1e-3)
    wu_u = orc.random_volume(r, sh + (3,), -0.02, 0.02)
    z = np.zeros(sh + (3,))
    g.update({"wu_g": wu_g, "wu_u": wu_u})
    for world in (1, 3):
        u1, a1, b1 = ref.warp_update(wu_g, wu_u, z, z, 0.01, 1, world=world)
        u2, a2, b2 = ref.warp_update(0.5 * wu_g, u1, a1, b1, 0.01, 2, world=world)
        g.update({f"wu_H{world}_u1": u1, f"wu_H{world}_m1": a1, f"wu_H{world}_v1": b1, f"wu_H{world}_u2": u2,
                  f"wu_H{world}_m2": a2, f"wu_H{world}_v2": b2})

    # --- multi-scale plumbing (resample.hpp:48-146, registration.hpp:100-115)
    rv = orc.random_volume(orc.rng(801), (13, 17, 19), 0.0, 2.0)
    g["rs_v"] = rv
    for f in (0.5, 0.25, 0.37, 2.0):
        g[f"rs_scale_{f}"] = ref.resample_scale(rv, f)
    rw = orc.random_volume(orc.rng(802), (7, 9, 11, 3), -0.1, 0.1)
    g["rs_w"] = rw
    for sh in ((13, 17, 19), (4, 5, 6), (1, 9, 11)):
        g["rs_warp_" + "x".join(map(str, sh))] = ref.resample_warp(rw, sh)
    g["rs_norm"] = ref.normalize(rv)

    # --- affine stage (registration.hpp:176-219) and the deformable stage (230-331), H = 1
    #     and H = 3, on the MI fixture; the Jacobian sign fraction (metrics.hpp:145-176)
    si = step_inputs(orc, (18, 20, 22), seed=4242, loss="mi")
    for loss in ("mse", "lncc", "mi"):
        A, t, tr = ref.affine_stage(si.f, si.m, [(2, 3), (1, 3)], lr=0.01, loss=loss)
        g.update({f"aff_{loss}_A": A, f"aff_{loss}_t": t, f"aff_{loss}_trace": tr})
    for loss, kind in (("lncc", "gaussian"), ("mi", "bspline3"), ("mi", "gaussian")):
        sl = step_inputs(orc, (18, 20, 22), seed=4242, loss=loss)
        for world in (1, 3):
            w, tr = ref.deformable_stage(sl.f, sl.m, [(2, 3), (1, 3)], sl.A, sl.t, loss=loss, mi_kind=kind,
                                         world=world)
            g.update({f"def_{loss}_{kind}_H{world}_warp": w, f"def_{loss}_{kind}_H{world}_trace": tr})
    jw = orc.random_volume(orc.rng(901), (8, 9, 10, 3), -0.4, 0.4)
    g.update({"jac_w": jw, "jac_frac": np.array(ref.jacobian_positive(jw))})

    # --- label evaluation (metrics.hpp:44-201) and nearest-neighbour label warping
    #     (sampler.hpp:331-365) on two overlapping ellipsoid maps
    la, lb = label_maps((7, 7, 6), (12, 5, 4)), label_maps((9, 8, 7), (11, 6, 5))
    lu = orc.random_volume(orc.rng(903), (14, 16, 18, 3), -0.2, 0.2)
    lA = np.eye(3) + orc.random_volume(orc.rng(904), (3, 3, 1), -0.03, 0.03).reshape(3, 3)
    lt = orc.random_volume(orc.rng(905), (3, 1, 1), -0.03, 0.03).reshape(3)
    lw = ref.warp_labels_nn(lb, lu, lA, lt)
    g.update({"lab_a": la, "lab_b": lb, "lab_u": lu, "lab_A": lA, "lab_t": lt, "lab_warped": lw,
              "lab_metrics": np.array(ref.label_metrics(la, lb)),
              "lab_metrics_sp": np.array(ref.label_metrics(la, lw, (0.7, 1.3, 2.1)))})

    # --- NIfTI-1 / raw + JSON IO (nifti.hpp), written and parsed by the reference itself
    g.update(nifti_fixtures(orc))

    path = os.path.join(OUT, "voxreg_golden.npz")
    np.savez_compressed(path, **g)
    print(f"wrote {path}: {len(g)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
