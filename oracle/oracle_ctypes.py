"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers declared in
oracle/oracle_api.h --
  prefix "arfr_": oracle/_ref/libarf_ref.so, the unmodified reference compiled in place;
  prefix "arfo_": oracle/_build/libarf_oracle.so, our C restatement (arf_oracle.c).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libarf_ref.so"
ORACLE_LIB = HERE / "_build" / "libarf_oracle.so"

MAXB = 32
MAXR = 8

dp = C.POINTER(C.c_double)
fp = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)


class Skel(C.Structure):
    _fields_ = [("n_bones", C.c_int), ("parent", C.c_int * MAXB), ("head", (C.c_double * 3) * MAXB),
                ("tail", (C.c_double * 3) * MAXB), ("radius", C.c_double * MAXB)]


class Figure(C.Structure):
    _fields_ = [("skel", Skel), ("color", (C.c_double * 3) * MAXB), ("amplitude", C.c_double * MAXB),
                ("softness", C.c_double)]


class LossCfg(C.Structure):
    _fields_ = [("w_rgb", C.c_double), ("w_alpha", C.c_double), ("w_hard", C.c_double), ("w_density", C.c_double),
                ("huber_delta", C.c_double)]


class AdamCfg(C.Structure):
    _fields_ = [("lr_grid", C.c_double), ("lr_mlp", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("total_steps", C.c_int64), ("final_lr_factor", C.c_double)]


class GridCfg(C.Structure):
    _fields_ = [("levels", C.c_int), ("features_per_level", C.c_int), ("table_size_log2", C.c_int),
                ("base_resolution", C.c_int), ("max_resolution", C.c_int), ("box_lo", C.c_double * 3),
                ("box_hi", C.c_double * 3)]


class MlpCfg(C.Structure):
    _fields_ = [("input_dim", C.c_int), ("hidden_dim", C.c_int), ("hidden_layers", C.c_int),
                ("output_dim", C.c_int)]


class Cam(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int), ("height", C.c_int), ("extrinsic", C.c_double * 12)]


class OccCfg(C.Structure):
    _fields_ = [("resolution", C.c_int), ("alpha_threshold", C.c_double), ("dilation", C.c_int),
                ("decay", C.c_double), ("update_interval", C.c_int)]


class Opts(C.Structure):
    _fields_ = [("samples_per_ray", C.c_int), ("stratified", C.c_int), ("epsilon_terminate", C.c_double),
                ("seed", C.c_uint64), ("frame_id", C.c_uint64)]


class Model(C.Structure):
    _fields_ = [("skel", Skel), ("grid", GridCfg), ("mlp", MlpCfg), ("skin_res", C.c_int * 3),
                ("skin_lo", C.c_double * 3), ("skin_hi", C.c_double * 3), ("canon_lo", C.c_double * 3),
                ("canon_hi", C.c_double * 3), ("norm_lo", C.c_double * 3), ("norm_hi", C.c_double * 3),
                ("max_iterations", C.c_int), ("tolerance", C.c_double), ("dedup_radius", C.c_double),
                ("grid_params", fp), ("n_grid", C.c_size_t), ("mlp_params", fp), ("n_mlp", C.c_size_t),
                ("skin_weights", dp), ("n_skin", C.c_size_t)]


class OccGrid(C.Structure):
    _fields_ = [("res", C.c_int * 3), ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3),
                ("density_threshold", C.c_double), ("dilation", C.c_int), ("values", fp), ("mask", u8p)]


class Trace(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("n_samples", C.c_int64), ("ray_first", i32p), ("ray_count", i32p),
                ("ray_hit", u8p), ("t_near", dp), ("t_far", dp), ("terminated_at", i32p), ("s_ray", i32p),
                ("s_index", i32p), ("s_has_root", u8p), ("s_density", fp), ("s_color", fp),
                ("s_canonical", dp), ("s_t", dp), ("s_delta", dp)]


def _p(a, t):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(t))


def build(which: str = "all") -> None:
    """make -C oracle (reference part only where /root/reference exists)."""
    have_ref = Path("/root/reference/proj/include/arf").is_dir()
    targets = {"all": ["oracle"] + (["ref", "adapter"] if have_ref else []),
               "oracle": ["oracle"], "ref": ["ref"], "adapter": ["adapter"]}[which]
    for t in targets:
        subprocess.run(["make", "-s", "-C", str(HERE), t], check=True)


class Checker:
    """One of the two CPU checkers; all methods take/return numpy arrays."""

    def __init__(self, kind: str = "ref"):
        self.kind = kind
        path = REF_LIB if kind == "ref" else ORACLE_LIB
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle {'ref' if kind == 'ref' else 'oracle'})")
        self.lib = C.CDLL(str(path))
        self.pre = "arfr_" if kind == "ref" else "arfo_"
        self._keep = []

    def f(self, name):
        fn = getattr(self.lib, self.pre + name)
        return fn

    def check(self, code):
        if code != 0:
            msg = self.f("last_error")
            msg.restype = C.c_char_p
            raise RuntimeError(f"{self.kind} checker error {code}: {msg().decode()}")

    # ---- structs from product-side python values
    @staticmethod
    def skel(sk) -> Skel:
        s = Skel()
        s.n_bones = len(sk.bones)
        for i, b in enumerate(sk.bones):
            s.parent[i] = b.parent
            for a in range(3):
                s.head[i][a] = b.head[a]
                s.tail[i][a] = b.tail[a]
            s.radius[i] = b.radius
        return s

    @staticmethod
    def grid(g) -> GridCfg:
        return GridCfg(g.levels, g.features_per_level, g.table_size_log2, g.base_resolution, g.max_resolution,
                       (C.c_double * 3)(*g.bounding_box.lo), (C.c_double * 3)(*g.bounding_box.hi))

    @staticmethod
    def mlp(m) -> MlpCfg:
        return MlpCfg(m.input_dim, m.hidden_dim, m.hidden_layers, m.output_dim)

    @staticmethod
    def cam(c) -> Cam:
        return Cam(c.fx, c.fy, c.cx, c.cy, c.width, c.height, (C.c_double * 12)(*[float(v) for v in c.extrinsic]))

    @staticmethod
    def opts(o) -> Opts:
        return Opts(o.samples_per_ray, int(bool(o.stratified)), o.epsilon_terminate, o.seed, o.frame_id)

    @staticmethod
    def occcfg(o) -> OccCfg:
        return OccCfg(o.resolution, o.alpha_threshold, o.dilation, o.decay, o.update_interval)

    # ---- model
    def build_model(self, sk, gcfg, mcfg, skin_res=(32, 32, 32), seed=0) -> Model:
        s, g, m = self.skel(sk), self.grid(gcfg), self.mlp(mcfg)
        res = (C.c_int * 3)(*skin_res)
        ng, nm, ns = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self.check(self.f("model_sizes")(C.byref(s), C.byref(g), C.byref(m), res, C.byref(ng), C.byref(nm),
                                         C.byref(ns)))
        M = Model()
        gp = np.zeros(ng.value, np.float32)
        mp = np.zeros(nm.value, np.float32)
        sw = np.zeros(ns.value, np.float64)
        M.grid_params, M.n_grid = _p(gp, C.c_float), ng.value
        M.mlp_params, M.n_mlp = _p(mp, C.c_float), nm.value
        M.skin_weights, M.n_skin = _p(sw, C.c_double), ns.value
        self.check(self.f("build_model")(C.byref(s), C.byref(g), C.byref(m), res, C.c_uint64(seed), C.byref(M)))
        M._arrays = (gp, mp, sw)  # keep alive
        return M

    @staticmethod
    def arrays(M: Model):
        return M._arrays

    @staticmethod
    def model_from_arrays(template: Model, grid_params, mlp_params, skin_weights) -> Model:
        M = Model()
        C.pointer(M)[0] = template
        gp = np.ascontiguousarray(grid_params, np.float32)
        mp = np.ascontiguousarray(mlp_params, np.float32)
        sw = np.ascontiguousarray(skin_weights, np.float64)
        M.grid_params, M.n_grid = _p(gp, C.c_float), gp.size
        M.mlp_params, M.n_mlp = _p(mp, C.c_float), mp.size
        M.skin_weights, M.n_skin = _p(sw, C.c_double), sw.size
        M._arrays = (gp, mp, sw)
        return M

    def level_resolutions(self, gcfg):
        out = np.zeros(gcfg.levels, np.int32)
        self.check(self.f("level_resolutions")(C.byref(self.grid(gcfg)), _p(out, C.c_int32)))
        return out.tolist()

    def hash_index(self, gcfg, level, cx, cy, cz):
        fn = self.f("hash_index")
        fn.restype = C.c_uint32
        return int(fn(C.byref(self.grid(gcfg)), int(level), int(cx), int(cy), int(cz)))

    def pose_from_joint_rotations(self, sk, rot9, g12):
        rot = np.ascontiguousarray(rot9, np.float64).reshape(-1, 9)
        g = np.ascontiguousarray(g12, np.float64).reshape(12)
        out = np.zeros((len(sk.bones), 12), np.float64)
        self.check(self.f("pose_from_joint_rotations")(C.byref(self.skel(sk)), _p(rot, C.c_double),
                                                       _p(g, C.c_double), _p(out, C.c_double)))
        return out

    def look_at(self, eye, target, up, focal, w, h):
        c = Cam()
        e, t, u = (np.asarray(v, np.float64) for v in (eye, target, up))
        self.check(self.f("look_at")(_p(e, C.c_double), _p(t, C.c_double), _p(u, C.c_double), C.c_double(focal),
                                     w, h, C.byref(c)))
        return c

    def skinning_weights(self, M, pts):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        w = np.zeros((p.shape[0], M.skel.n_bones), np.float64)
        self.check(self.f("skinning_weights")(C.byref(M), _p(p, C.c_double), C.c_int64(p.shape[0]),
                                              _p(w, C.c_double)))
        return w

    def inverse_lbs(self, M, bones12, pre12, cutoff, pts):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        b = np.ascontiguousarray(bones12, np.float64)
        pr = np.ascontiguousarray(pre12, np.float64)
        n = p.shape[0]
        cnt = np.zeros(n, np.int32)
        roots = np.zeros((n, MAXR, 3), np.float64)
        res = np.zeros((n, MAXR), np.float64)
        self.check(self.f("inverse_lbs")(C.byref(M), _p(b, C.c_double), _p(pr, C.c_double), C.c_double(cutoff),
                                         _p(p, C.c_double), C.c_int64(n), _p(cnt, C.c_int32),
                                         _p(roots, C.c_double), _p(res, C.c_double)))
        return cnt, roots, res

    def hash_encode(self, M, pts):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        D = M.grid.levels * M.grid.features_per_level
        out = np.zeros((p.shape[0], D), np.float32)
        self.check(self.f("hash_encode")(C.byref(M), _p(p, C.c_double), C.c_int64(p.shape[0]), _p(out, C.c_float)))
        return out

    def field_query(self, M, pts):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        d = np.zeros(p.shape[0], np.float32)
        c = np.zeros((p.shape[0], 3), np.float32)
        self.check(self.f("field_query")(C.byref(M), _p(p, C.c_double), C.c_int64(p.shape[0]), _p(d, C.c_float),
                                         _p(c, C.c_float)))
        return d, c

    def posed_query(self, M, bones12, global12, pts):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        n = p.shape[0]
        d = np.zeros(n, np.float32)
        c = np.zeros((n, 3), np.float32)
        x = np.zeros((n, 3), np.float64)
        h = np.zeros(n, np.uint8)
        b = np.ascontiguousarray(bones12, np.float64)
        g = np.ascontiguousarray(global12, np.float64)
        self.check(self.f("posed_query")(C.byref(M), _p(b, C.c_double), _p(g, C.c_double), _p(p, C.c_double),
                                         C.c_int64(n), _p(d, C.c_float), _p(c, C.c_float), _p(x, C.c_double),
                                         _p(h, C.c_uint8)))
        return d, c, x, h.astype(bool)

    def _occ(self, res):
        n = res ** 3
        v = np.zeros(n, np.float32)
        m = np.zeros(n, np.uint8)
        g = OccGrid()
        g.values, g.mask = _p(v, C.c_float), _p(m, C.c_uint8)
        g._arrays = (v, m)
        return g

    def occ_empty(self, lo, hi, cfg):
        g = self._occ(cfg.resolution)
        lo_ = np.asarray(lo, np.float64)
        hi_ = np.asarray(hi, np.float64)
        self.check(self.f("occ_empty")(_p(lo_, C.c_double), _p(hi_, C.c_double), C.byref(self.occcfg(cfg)),
                                       C.byref(g)))
        return g

    def build_inference_grid(self, M, bones12, global12, cfg):
        g = self._occ(cfg.resolution)
        cnt = np.zeros(2, np.uint64)
        b = np.ascontiguousarray(bones12, np.float64)
        gl = np.ascontiguousarray(global12, np.float64)
        self.check(self.f("build_inference_grid")(C.byref(M), _p(b, C.c_double), _p(gl, C.c_double),
                                                  C.byref(self.occcfg(cfg)), C.byref(g), _p(cnt, C.c_uint64)))
        return g, cnt

    def update_training_grid(self, M, bones12_list, global12_list, decay, seed, step, g):
        b = np.ascontiguousarray(np.stack(bones12_list), np.float64)
        gl = np.ascontiguousarray(np.stack(global12_list), np.float64)
        cnt = np.zeros(2, np.uint64)
        self.check(self.f("update_training_grid")(C.byref(M), len(bones12_list), _p(b, C.c_double),
                                                  _p(gl, C.c_double), C.c_double(decay), C.c_uint64(seed),
                                                  C.c_uint64(step), C.byref(g), _p(cnt, C.c_uint64)))
        return cnt

    def occ_rebuild_mask(self, g):
        self.check(self.f("occ_rebuild_mask")(C.byref(g)))

    @staticmethod
    def occ_arrays(g):
        return g._arrays

    def figure(self, fig) -> Figure:
        f = Figure()
        f.skel = self.skel(fig.skeleton)
        col = np.asarray(fig.colors, np.float64).reshape(-1, 3)
        amp = np.asarray(fig.amplitudes, np.float64).reshape(-1)
        for i in range(col.shape[0]):
            for c in range(3):
                f.color[i][c] = float(col[i, c])
            f.amplitude[i] = float(amp[i])
        f.softness = float(fig.softness)
        return f

    def figure_query(self, fig, pts, bones12=None):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        dens = np.zeros(p.shape[0], np.float64)
        col = np.zeros((p.shape[0], 3), np.float64)
        b = None if bones12 is None else np.ascontiguousarray(bones12, np.float64)
        self.check(self.f("figure_query")(C.byref(self.figure(fig)), _p(b, C.c_double), _p(p, C.c_double),
                                          C.c_int64(p.shape[0]), _p(dens, C.c_double), _p(col, C.c_double)))
        return dens, col

    def figure_render(self, fig, bones12, global12, lo, hi, cam, opts):
        W, H = cam.width, cam.height
        rgb = np.zeros((H, W, 3), np.float32)
        alpha = np.zeros((H, W), np.float32)
        mask = np.zeros((H, W), np.uint8)
        b = np.ascontiguousarray(bones12, np.float64)
        g = np.ascontiguousarray(global12, np.float64)
        lo = np.ascontiguousarray(lo, np.float64)
        hi = np.ascontiguousarray(hi, np.float64)
        self.check(self.f("figure_render")(C.byref(self.figure(fig)), _p(b, C.c_double), _p(g, C.c_double),
                                           _p(lo, C.c_double), _p(hi, C.c_double), C.byref(self.cam(cam)),
                                           C.byref(self.opts(opts)), _p(rgb, C.c_float), _p(alpha, C.c_float),
                                           _p(mask, C.c_uint8)))
        return rgb, alpha, mask

    # ---- training pieces with no reference code: oracle restatement only
    def losses(self, rgb, alpha, gt_rgb, gt_alpha, cfg):
        assert self.kind == "oracle", "losses exist only in the C restatement (the reference has none)"
        r = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
        n = r.shape[0]
        a = np.ascontiguousarray(alpha, np.float32).reshape(n)
        gr = np.ascontiguousarray(gt_rgb, np.float32).reshape(n, 3)
        ga = np.ascontiguousarray(gt_alpha, np.float32).reshape(n)
        l4 = np.zeros(4, np.float64)
        dr = np.zeros((n, 3), np.float32)
        da = np.zeros(n, np.float32)
        c = LossCfg(cfg.w_rgb, cfg.w_alpha, cfg.w_hard, cfg.w_density, cfg.huber_delta)
        self.check(self.f("losses")(C.c_int64(n), _p(r, C.c_float), _p(a, C.c_float), _p(gr, C.c_float),
                                    _p(ga, C.c_float), C.byref(c), _p(l4, C.c_double), _p(dr, C.c_float),
                                    _p(da, C.c_float)))
        return l4, dr, da

    def adam(self, p, g, m, v, cfg, step, mlp_offset):
        """In place on float32 numpy arrays (one Adam step, grads zeroed)."""
        assert self.kind == "oracle"
        for a in (p, g, m, v):
            assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
        c = AdamCfg(cfg.lr_grid, cfg.lr_mlp, cfg.beta1, cfg.beta2, cfg.eps, int(cfg.total_steps), cfg.final_lr_factor)
        self.check(self.f("adam")(C.c_int64(p.size), _p(p, C.c_float), _p(g, C.c_float), _p(m, C.c_float),
                                  _p(v, C.c_float), C.byref(c), C.c_int64(step), C.c_int64(mlp_offset)))

    def render(self, M, bones12, global12, cam, occ, opts):
        W, H = cam.width, cam.height
        rgb = np.zeros((H, W, 3), np.float32)
        alpha = np.zeros((H, W), np.float32)
        cnt = np.zeros(2, np.uint64)
        b = np.ascontiguousarray(bones12, np.float64)
        g = np.ascontiguousarray(global12, np.float64)
        self.check(self.f("render")(C.byref(M), _p(b, C.c_double), _p(g, C.c_double), C.byref(self.cam(cam)),
                                    C.byref(occ) if occ is not None else None, C.byref(self.opts(opts)),
                                    _p(rgb, C.c_float), _p(alpha, C.c_float), _p(cnt, C.c_uint64)))
        return rgb, alpha, cnt

    def render_trace(self, M, bones12, global12, cam, occ, opts, capacity=None):
        W, H = cam.width, cam.height
        npix = W * H
        cap = capacity or npix * opts.samples_per_ray
        rgb = np.zeros((H, W, 3), np.float32)
        alpha = np.zeros((H, W), np.float32)
        cnt = np.zeros(2, np.uint64)
        arr = dict(ray_first=np.zeros(npix, np.int32), ray_count=np.zeros(npix, np.int32),
                   ray_hit=np.zeros(npix, np.uint8), t_near=np.zeros(npix), t_far=np.zeros(npix),
                   terminated_at=np.zeros(npix, np.int32), s_ray=np.zeros(cap, np.int32),
                   s_index=np.zeros(cap, np.int32), s_has_root=np.zeros(cap, np.uint8),
                   s_density=np.zeros(cap, np.float32), s_color=np.zeros((cap, 3), np.float32),
                   s_canonical=np.zeros((cap, 3)), s_t=np.zeros(cap), s_delta=np.zeros(cap))
        tr = Trace()
        tr.capacity = cap
        types = {np.dtype(np.int32): C.c_int32, np.dtype(np.uint8): C.c_uint8, np.dtype(np.float64): C.c_double,
                 np.dtype(np.float32): C.c_float}
        for k, a in arr.items():
            setattr(tr, k, _p(a, types[a.dtype]))
        b = np.ascontiguousarray(bones12, np.float64)
        g = np.ascontiguousarray(global12, np.float64)
        self.check(self.f("render_trace")(C.byref(M), _p(b, C.c_double), _p(g, C.c_double), C.byref(self.cam(cam)),
                                          C.byref(occ) if occ is not None else None, C.byref(self.opts(opts)),
                                          _p(rgb, C.c_float), _p(alpha, C.c_float), _p(cnt, C.c_uint64),
                                          C.byref(tr)))
        n = tr.n_samples
        for k in list(arr):
            if k.startswith("s_"):
                arr[k] = arr[k][:n]
        arr["n_samples"] = n
        return rgb, alpha, cnt, arr

    def composite(self, ray_t, ray_delta, ray_skip, ray_dens, ray_col, eps):
        t = np.ascontiguousarray(ray_t, np.float64)
        n = t.shape[0]
        d = np.ascontiguousarray(ray_delta, np.float64)
        s = np.ascontiguousarray(ray_skip, np.uint8)
        de = np.ascontiguousarray(ray_dens, np.float32)
        co = np.ascontiguousarray(ray_col, np.float32)
        c3 = np.zeros(3)
        a = C.c_double()
        term = C.c_int()
        self.check(self.f("composite")(n, _p(t, C.c_double), _p(d, C.c_double), _p(s, C.c_uint8),
                                       _p(de, C.c_float), _p(co, C.c_float), C.c_double(eps), _p(c3, C.c_double),
                                       C.byref(a), C.byref(term)))
        return c3, a.value, term.value

    def composite_backward(self, ray_t, ray_delta, ray_skip, ray_dens, ray_col, eps, dC, dA):
        t = np.ascontiguousarray(ray_t, np.float64)
        n = t.shape[0]
        d = np.ascontiguousarray(ray_delta, np.float64)
        s = np.ascontiguousarray(ray_skip, np.uint8)
        de = np.ascontiguousarray(ray_dens, np.float32)
        co = np.ascontiguousarray(ray_col, np.float32)
        dc = np.ascontiguousarray(dC, np.float64)
        ds = np.zeros(n)
        dcs = np.zeros((n, 3))
        self.check(self.f("composite_backward")(n, _p(t, C.c_double), _p(d, C.c_double), _p(s, C.c_uint8),
                                                _p(de, C.c_float), _p(co, C.c_float), C.c_double(eps),
                                                _p(dc, C.c_double), C.c_double(dA), _p(ds, C.c_double),
                                                _p(dcs, C.c_double)))
        return ds, dcs

    def field_query_backward(self, M, pts, d_dens, d_col, grid_grad=None, mlp_grad=None):
        p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        dd = np.ascontiguousarray(d_dens, np.float32)
        dc = np.ascontiguousarray(d_col, np.float32)
        gg = np.zeros(M.n_grid, np.float32) if grid_grad is None else grid_grad
        mg = np.zeros(M.n_mlp, np.float32) if mlp_grad is None else mlp_grad
        self.check(self.f("field_query_backward")(C.byref(M), _p(p, C.c_double), C.c_int64(p.shape[0]),
                                                  _p(dd, C.c_float), _p(dc, C.c_float), _p(gg, C.c_float),
                                                  _p(mg, C.c_float)))
        return gg, mg

    def train_fwd_bwd(self, M, bones12, global12, cam, occ, opts, px, py, d_color, d_alpha):
        n = len(px)
        pxa = np.ascontiguousarray(px, np.int32)
        pya = np.ascontiguousarray(py, np.int32)
        dc = np.ascontiguousarray(d_color, np.float32)
        da = np.ascontiguousarray(d_alpha, np.float32)
        rgb = np.zeros((n, 3), np.float32)
        alpha = np.zeros(n, np.float32)
        gg = np.zeros(M.n_grid, np.float32)
        mg = np.zeros(M.n_mlp, np.float32)
        cnt = np.zeros(2, np.uint64)
        b = np.ascontiguousarray(bones12, np.float64)
        g = np.ascontiguousarray(global12, np.float64)
        self.check(self.f("train_fwd_bwd")(C.byref(M), _p(b, C.c_double), _p(g, C.c_double), C.byref(self.cam(cam)),
                                           C.byref(occ) if occ is not None else None, C.byref(self.opts(opts)),
                                           C.c_int64(n), _p(pxa, C.c_int32), _p(pya, C.c_int32), _p(dc, C.c_float),
                                           _p(da, C.c_float), _p(rgb, C.c_float), _p(alpha, C.c_float),
                                           _p(gg, C.c_float), _p(mg, C.c_float), _p(cnt, C.c_uint64)))
        return rgb, alpha, gg, mg, cnt

    def bench_frames(self, M, poses, cam, occ_cfg, opts, keep_last: bool = False):
        """reference-only: time n x (inference grid + render) with its own thread pool.
        keep_last: also return the last frame's (rgb, alpha, occupancy mask)."""
        assert self.kind == "ref"
        n = len(poses)
        b = np.ascontiguousarray(np.stack([p.bone_transforms for p in poses]), np.float64)
        g = np.ascontiguousarray(np.stack([p.global_transform for p in poses]), np.float64)
        secs = np.zeros(n)
        posed = np.zeros(n, np.uint64)
        last = None
        if keep_last:
            res = occ_cfg.resolution
            last = (np.zeros((cam.height, cam.width, 3), np.float32), np.zeros((cam.height, cam.width), np.float32),
                    np.zeros(res ** 3, np.uint8))
        self.check(self.f("bench_frames")(C.byref(M), n, _p(b, C.c_double), _p(g, C.c_double),
                                          C.byref(self.cam(cam)), C.byref(self.occcfg(occ_cfg)),
                                          C.byref(self.opts(opts)), _p(secs, C.c_double), _p(posed, C.c_uint64),
                                          *((None, None, None) if last is None else
                                            (_p(last[0], C.c_float), _p(last[1], C.c_float),
                                             _p(last[2], C.c_uint8)))))
        return (secs, posed, last) if keep_last else (secs, posed)

    def random_pose(self, sk, seed, stream=7, max_angle=0.5, yaw=0.3):
        """reference-only: (bones12[n,12], global12[12]) of the fixture pose built by the reference
        (ref_driver.cpp arfr_random_pose; fixtures.random_pose restates it)."""
        assert self.kind == "ref"
        nb = len(sk.bones)
        b = np.zeros((nb, 12), np.float64)
        g = np.zeros(12, np.float64)
        self.check(self.f("random_pose")(C.byref(self.skel(sk)), C.c_uint64(seed), C.c_uint64(stream),
                                         C.c_double(max_angle), C.c_double(yaw), _p(b, C.c_double),
                                         _p(g, C.c_double)))
        return b, g

    def default_camera(self, sk, w, h) -> Cam:
        """reference-only: arf::default_camera (R/scene.hpp:190-197)."""
        assert self.kind == "ref"
        c = Cam()
        self.check(self.f("default_camera")(C.byref(self.skel(sk)), int(w), int(h), C.byref(c)))
        return c

    def thread_count(self):
        return int(self.f("thread_count")())
