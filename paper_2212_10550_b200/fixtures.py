"""Deterministic synthetic workloads of BASELINE.json's configs.

All draws use the reference's keyed PCG32 streams (R/rng.hpp) restated in Python
integers, one statement per draw in the order SURVEY.md §8d pins. Rotation /
rigid algebra keeps the reference's operand order (R/math.hpp) so the poses and
cameras are bit-identical to the ones the reference would build.
"""
from __future__ import annotations

import math

import numpy as np

from .arf import (Bone, Camera, HashGridConfig, MlpConfig, OccupancyConfig, RenderOptions, Skeleton,
                  SkeletonPose, pose_from_joint_rotations)

M64 = (1 << 64) - 1
PCG_MULT = 6364136223846793005


def splitmix64(x: int) -> int:  # R/rng.hpp:7-12
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix_key(a: int, b: int = 0, c: int = 0, d: int = 0) -> int:  # R/rng.hpp:14-20
    h = splitmix64(a & M64)
    h = splitmix64(h ^ (b & M64))
    h = splitmix64(h ^ (c & M64))
    h = splitmix64(h ^ (d & M64))
    return h


class Pcg32:  # R/rng.hpp:24-58
    def __init__(self, seed: int, seq: int):
        self.state = 0
        self.inc = ((seq << 1) | 1) & M64
        self.next_u32()
        self.state = (self.state + seed) & M64
        self.next_u32()

    def next_u32(self) -> int:
        old = self.state
        self.state = (old * PCG_MULT + self.inc) & M64
        xorshifted = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        return ((xorshifted >> rot) | (xorshifted << ((32 - rot) & 31))) & 0xFFFFFFFF

    def next_double(self) -> float:
        return self.next_u32() * 2.0 ** -32

    def next_below(self, n: int) -> int:
        return (self.next_u32() * n) >> 32

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()


def keyed_rng(seed: int, a: int, b: int = 0, c: int = 0) -> Pcg32:  # R/rng.hpp:61-63
    return Pcg32(mix_key(seed, a, b), mix_key(c, a ^ 0x5851F42D4C957F2D, seed))


def pcg_stream_u32(rng: Pcg32, count: int) -> np.ndarray:
    """The next `count` outputs of `rng` (vectorised; identical to calling next_u32 in a
    loop). State k = A_k*s0 + inc*S_k (mod 2^64), A_k = mult^k, S_k = sum_{j<k} mult^j."""
    with np.errstate(over="ignore"):
        mult = np.full(count, PCG_MULT, np.uint64)
        mult[0] = 1
        A = np.cumprod(mult, dtype=np.uint64)              # mult^k, wraps mod 2^64
        S = np.concatenate([np.zeros(1, np.uint64), np.cumsum(A[:-1], dtype=np.uint64)])
        old = A * np.uint64(rng.state) + S * np.uint64(rng.inc)
        xs = (((old >> np.uint64(18)) ^ old) >> np.uint64(27)) & np.uint64(0xFFFFFFFF)
        rot = old >> np.uint64(59)
        out = ((xs >> rot) | (xs << ((np.uint64(32) - rot) & np.uint64(31)))) & np.uint64(0xFFFFFFFF)
    # advance the Python generator past the consumed draws
    st = rng.state
    a_n, s_n = int(A[-1]) * PCG_MULT % (1 << 64), (int(S[-1]) + int(A[-1])) % (1 << 64)
    rng.state = (a_n * st + s_n * rng.inc) % (1 << 64)
    return out.astype(np.uint64)


# ---- rotation helpers (R/math.hpp:160-173, :210-212) -------------------------

def axis_angle(a, angle: float) -> np.ndarray:
    ax, ay, az = float(a[0]), float(a[1]), float(a[2])
    c = math.cos(angle)
    s = math.sin(angle)
    t = 1.0 - c
    return np.array([t * ax * ax + c, t * ax * ay - s * az, t * ax * az + s * ay,
                     t * ax * ay + s * az, t * ay * ay + c, t * ay * az - s * ax,
                     t * ax * az - s * ay, t * ay * az + s * ax, t * az * az + c], np.float64)


def rot_x(a):
    return axis_angle((1.0, 0.0, 0.0), a)


def rot_y(a):
    return axis_angle((0.0, 1.0, 0.0), a)


def rot_z(a):
    return axis_angle((0.0, 0.0, 1.0), a)


def about_point(pivot, r9) -> np.ndarray:
    """Rigid::about_point: {R, pivot - R*pivot}."""
    m = r9
    px, py, pz = (float(v) for v in pivot)
    rp = (m[0] * px + m[1] * py + m[2] * pz, m[3] * px + m[4] * py + m[5] * pz, m[6] * px + m[7] * py + m[8] * pz)
    out = np.zeros(12, np.float64)
    out[:9] = m
    out[9:] = (px - rp[0], py - rp[1], pz - rp[2])
    return out


def yaw_about(pivot, yaw: float) -> np.ndarray:  # R/scene.hpp:169-171
    return about_point(pivot, rot_y(yaw))


IDENTITY9 = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1], np.float64)


# ---- skeletons ----------------------------------------------------------------

_SMPL24_PARENTS = [-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21]
_SMPL24_JOINTS = [(0, .95, 0), (.09, .88, 0), (-.09, .88, 0), (0, 1.05, 0), (.11, .50, 0), (-.11, .50, 0),
                  (0, 1.18, 0), (.12, .09, 0), (-.12, .09, 0), (0, 1.24, 0), (.13, .03, .12), (-.13, .03, .12),
                  (0, 1.45, 0), (.07, 1.38, 0), (-.07, 1.38, 0), (0, 1.55, .02), (.18, 1.40, 0), (-.18, 1.40, 0),
                  (.45, 1.40, 0), (-.45, 1.40, 0), (.70, 1.40, 0), (-.70, 1.40, 0), (.78, 1.40, 0), (-.78, 1.40, 0)]
_SMPL24_CHILD = [3, 4, 5, 6, 7, 8, 9, 10, 11, 12, -1, -1, 15, 16, 17, -1, 18, 19, 20, 21, 22, 23, -1, -1]
_SMPL24_RADII = [.12, .08, .08, .12, .07, .07, .12, .05, .05, .12, .04, .04, .05, .05, .05, .09, .045, .045, .04,
                 .04, .035, .035, .03, .03]
_SMPL24_LEAF = {10: (0.0, 0.0, 0.08), 11: (0.0, 0.0, 0.08), 15: (0.0, 0.17, 0.0), 22: (0.08, 0.0, 0.0),
                23: (-0.08, 0.0, 0.0)}


def smpl24() -> Skeleton:
    """24-bone SMPL-like capsule skeleton."""
    bones = []
    for i in range(24):
        head = tuple(float(v) for v in _SMPL24_JOINTS[i])
        if _SMPL24_CHILD[i] >= 0:
            tail = tuple(float(v) for v in _SMPL24_JOINTS[_SMPL24_CHILD[i]])
        else:
            off = _SMPL24_LEAF[i]
            tail = (head[0] + off[0], head[1] + off[1], head[2] + off[2])
        bones.append(Bone(_SMPL24_PARENTS[i], head, tail, _SMPL24_RADII[i]))
    return Skeleton(bones)


def default_figure_skeleton(n_bones: int = 10) -> Skeleton:
    """The reference's 10-bone default_figure() skeleton (R/scene.hpp:129-154)."""
    spec = [(-1, (0.00, 0.95, 0.00), (0.00, 1.45, 0.00), 0.11), (0, (0.00, 1.47, 0.00), (0.00, 1.66, 0.00), 0.09),
            (0, (0.13, 1.38, 0.00), (0.38, 1.27, 0.00), 0.050), (2, (0.38, 1.27, 0.00), (0.62, 1.16, 0.00), 0.045),
            (0, (-0.13, 1.38, 0.00), (-0.38, 1.27, 0.00), 0.050), (4, (-0.38, 1.27, 0.00), (-0.62, 1.16, 0.00), 0.045),
            (0, (0.10, 0.92, 0.00), (0.13, 0.50, 0.00), 0.070), (6, (0.13, 0.50, 0.00), (0.15, 0.07, 0.00), 0.055),
            (0, (-0.10, 0.92, 0.00), (-0.13, 0.50, 0.00), 0.070), (8, (-0.13, 0.50, 0.00), (-0.15, 0.07, 0.00), 0.055)]
    return Skeleton([Bone(p, h, t, r) for (p, h, t, r) in spec[:n_bones]])


def default_figure():
    """The reference's default_figure() (R/scene.hpp:129-154): 10 colored capsules,
    amplitude 80, softness 0.012."""
    from .arf import CapsuleFigure
    colors = [(0.90, 0.10, 0.10), (0.95, 0.85, 0.10), (0.10, 0.80, 0.15), (0.10, 0.25, 0.90), (0.10, 0.85, 0.80),
              (0.85, 0.15, 0.85), (0.95, 0.55, 0.10), (0.55, 0.10, 0.85), (0.10, 0.55, 0.45), (0.60, 0.80, 0.10)]
    return CapsuleFigure(default_figure_skeleton(), np.array(colors), np.full(10, 80.0), 0.012)


def figure_for(skel: Skeleton, seed: int = 77, amplitude: float = 80.0, softness: float = 0.012):
    """A CapsuleFigure over any skeleton (e.g. smpl24): per-bone colors U(0.1, 0.95)^3 from
    keyed_rng(seed, 3), drawn r, g, b per bone in bone order."""
    from .arf import CapsuleFigure
    rng = keyed_rng(seed, 3)
    cols = np.array([[rng.uniform(0.1, 0.95) for _ in range(3)] for _ in range(skel.bone_count())])
    return CapsuleFigure(skel, cols, np.full(skel.bone_count(), amplitude), softness)


# ---- poses / cameras ----------------------------------------------------------

def random_pose(skel: Skeleton, seed: int, stream: int = 7, max_angle: float = 0.5, yaw: float = 0.3) -> SkeletonPose:
    """Per non-root joint: axis U(-1,1)^3 normalised, angle U(-a,a); global yaw about the root
    head (keyed_rng(42, 7), a = 0.5, yaw 0.3). Draw order: x, y, z, angle."""
    rng = keyed_rng(seed, stream)
    rots = [IDENTITY9.copy()]
    for _ in range(1, skel.bone_count()):
        ax = rng.uniform(-1.0, 1.0)
        ay = rng.uniform(-1.0, 1.0)
        az = rng.uniform(-1.0, 1.0)
        ang = rng.uniform(-max_angle, max_angle)
        n = math.sqrt(ax * ax + ay * ay + az * az)
        rots.append(axis_angle((ax / n, ay / n, az / n), ang))
    g = yaw_about(skel.bones[0].head, yaw)
    return pose_from_joint_rotations(skel, np.stack(rots), g)


def animation_poses(skel: Skeleton, n_frames: int = 100, base_seed: int = 1000) -> list:
    """Config 4: 100 novel poses random_pose(seed = 1000 + f), yaw sweeping with f."""
    return [random_pose(skel, base_seed + f, yaw=0.3 + 2.0 * math.pi * f / max(n_frames, 1))
            for f in range(n_frames)]


def default_camera(skel: Skeleton, width: int = 128, height: int = 128) -> Camera:  # R/scene.hpp:190-197
    h0 = skel.bones[0].head
    target = (h0[0] + 0.0, h0[1] + -0.05, h0[2] + 0.0)
    dist = 3.2
    eye = (target[0] + 0.0, target[1] + 0.0, target[2] + -dist)
    focal = height * dist / 2.3
    return Camera.look_at(eye, target, (0.0, 1.0, 0.0), focal, width, height)


def bend_pose_rotations(n_bones: int, elbow: float, knee: float) -> np.ndarray:  # R/scene.hpp:157-167
    rots = np.tile(IDENTITY9, (n_bones, 1))
    if n_bones >= 10:
        rots[3] = rot_z(elbow)
        rots[5] = rot_z(-elbow)
        rots[7] = rot_x(knee)
        rots[9] = rot_x(-knee)
    return rots


# ---- configs (BASELINE.json) -------------------------------------------------

def config1_grid() -> HashGridConfig:
    """16-level hash grid, 2^19 entries, F=2, N_min 16, N_max 2048 (SURVEY.md §8 intro)."""
    return HashGridConfig(levels=16, features_per_level=2, table_size_log2=19, base_resolution=16,
                          max_resolution=2048)


def config1_mlp() -> MlpConfig:
    return MlpConfig(input_dim=32, hidden_dim=64, hidden_layers=2, output_dim=4)


CONFIG1_SEED = 1234
CONFIG1_POSE_SEED = 42


def config1_render_options() -> RenderOptions:
    return RenderOptions(samples_per_ray=128, stratified=False, epsilon_terminate=1e-3, seed=0, frame_id=0)


def config1_occupancy() -> OccupancyConfig:
    return OccupancyConfig()


def microbench_pose(skel9: Skeleton) -> SkeletonPose:
    """Config 2: rot[2]=rot_z(-.3), rot[3]=rot_z(.6), rot[7]=rot_x(.5), global yaw 0.4."""
    rots = np.tile(IDENTITY9, (skel9.bone_count(), 1))
    rots[2] = rot_z(-0.3)
    rots[3] = rot_z(0.6)
    rots[7] = rot_x(0.5)
    return pose_from_joint_rotations(skel9, rots, yaw_about(skel9.bones[0].head, 0.4))


def microbench_points(skel9: Skeleton, pose: SkeletonPose, n: int, seed: int = 5, stream: int = 5) -> np.ndarray:
    """Config 2 points: keyed_rng(5,5); per point draw segment, u, then jitter x, y, z U(+-0.06)
    around the POSED segment B_i(head) + (B_i(tail) - B_i(head)) * u."""
    rng = keyed_rng(seed, stream)
    nb = skel9.bone_count()
    heads = np.array([_apply(pose.bone_transforms[i], b.head) for i, b in enumerate(skel9.bones)])
    tails = np.array([_apply(pose.bone_transforms[i], b.tail) for i, b in enumerate(skel9.bones)])
    d = pcg_stream_u32(rng, 5 * n).reshape(n, 5)
    seg = ((d[:, 0] * np.uint64(nb)) >> np.uint64(32)).astype(np.int64)      # next_below
    u = d[:, 1].astype(np.float64) * 2.0 ** -32                              # next_double
    span = 0.06 - (-0.06)
    j = -0.06 + span * (d[:, 2:5].astype(np.float64) * 2.0 ** -32)           # uniform(-.06, .06)
    a, b = heads[seg], tails[seg]
    return a + (b - a) * u[:, None] + j


def _apply(T, x):
    m = T
    return (m[0] * x[0] + m[1] * x[1] + m[2] * x[2] + m[9], m[3] * x[0] + m[4] * x[1] + m[5] * x[2] + m[10],
            m[6] * x[0] + m[7] * x[1] + m[8] * x[2] + m[11])
