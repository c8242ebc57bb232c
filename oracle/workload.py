"""TEST INFRASTRUCTURE ONLY: bench.py's workload (BASELINE configs[0]/[3]) restated for the
reference arm, built through the reference alone -- no import of the product package.

  smpl24 capsule skeleton
  animation poses             ref_driver.cpp arfr_random_pose: keyed_rng (R/rng.hpp:61-63),
                              Mat3d::axis_angle (R/math.hpp:170-178), yaw_about
                              (R/scene.hpp:169-171), pose_from_joint_rotations
                              (R/skeleton.hpp:93-110)
  camera                      arf::default_camera (R/scene.hpp:190-197)
  configs                     L16 F2 T19 16->2048, MLP 32-64-64-4, 32^3 skinning, 64^3
                              occupancy, N=128 midpoints

tests/test_oracle_cpu.py::test_reference_workload_matches_fixtures pins every pose and the
camera bit-for-bit to paper_2212_10550_b200.fixtures (the product arm's workload).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Bone:
    parent: int
    head: tuple
    tail: tuple
    radius: float


@dataclass
class Skeleton:
    bones: list


@dataclass
class Box:
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)


@dataclass
class GridConfig:  # R/hash_grid.hpp:12-32
    levels: int = 16
    features_per_level: int = 2
    table_size_log2: int = 19
    base_resolution: int = 16
    max_resolution: int = 2048
    bounding_box: Box = field(default_factory=Box)


@dataclass
class MlpConfig:  # R/mlp.hpp:11-23
    input_dim: int = 32
    hidden_dim: int = 64
    hidden_layers: int = 2
    output_dim: int = 4


@dataclass
class OccupancyConfig:  # R/occupancy.hpp:13-28
    resolution: int = 64
    alpha_threshold: float = 0.01
    dilation: int = 1
    decay: float = 0.95
    update_interval: int = 16


@dataclass
class RenderOptions:  # R/render.hpp:159-165
    samples_per_ray: int = 128
    stratified: bool = False
    epsilon_terminate: float = 1e-3
    seed: int = 0
    frame_id: int = 0


@dataclass
class Pose:
    bone_transforms: np.ndarray
    global_transform: np.ndarray


_PARENTS = [-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21]
_JOINTS = [(0, .95, 0), (.09, .88, 0), (-.09, .88, 0), (0, 1.05, 0), (.11, .50, 0), (-.11, .50, 0),
           (0, 1.18, 0), (.12, .09, 0), (-.12, .09, 0), (0, 1.24, 0), (.13, .03, .12), (-.13, .03, .12),
           (0, 1.45, 0), (.07, 1.38, 0), (-.07, 1.38, 0), (0, 1.55, .02), (.18, 1.40, 0), (-.18, 1.40, 0),
           (.45, 1.40, 0), (-.45, 1.40, 0), (.70, 1.40, 0), (-.70, 1.40, 0), (.78, 1.40, 0), (-.78, 1.40, 0)]
_CHILD = [3, 4, 5, 6, 7, 8, 9, 10, 11, 12, -1, -1, 15, 16, 17, -1, 18, 19, 20, 21, 22, 23, -1, -1]
_RADII = [.12, .08, .08, .12, .07, .07, .12, .05, .05, .12, .04, .04, .05, .05, .05, .09, .045, .045, .04,
          .04, .035, .035, .03, .03]
_LEAF = {10: (0.0, 0.0, 0.08), 11: (0.0, 0.0, 0.08), 15: (0.0, 0.17, 0.0), 22: (0.08, 0.0, 0.0),
         23: (-0.08, 0.0, 0.0)}

SEED = 1234          # build_model seed
SKIN_RES = (32, 32, 32)
N_FRAMES = 100


def smpl24() -> Skeleton:
    bones = []
    for i in range(24):
        head = tuple(float(v) for v in _JOINTS[i])
        if _CHILD[i] >= 0:
            tail = tuple(float(v) for v in _JOINTS[_CHILD[i]])
        else:
            o = _LEAF[i]
            tail = (head[0] + o[0], head[1] + o[1], head[2] + o[2])
        bones.append(Bone(_PARENTS[i], head, tail, _RADII[i]))
    return Skeleton(bones)


def animation_poses(ref, sk: Skeleton, n_frames: int = N_FRAMES, base_seed: int = 1000) -> list:
    """Config 4: random_pose(seed = 1000 + f, stream 7, angle 0.5), yaw 0.3 + 2 pi f / n."""
    out = []
    for f in range(n_frames):
        b, g = ref.random_pose(sk, base_seed + f, 7, 0.5, 0.3 + 2.0 * math.pi * f / max(n_frames, 1))
        out.append(Pose(b, g))
    return out


def build(ref, width: int = 540, height: int = 540):
    """(skeleton, reference model, poses, camera, occupancy config, render options)."""
    sk = smpl24()
    rm = ref.build_model(sk, GridConfig(), MlpConfig(), SKIN_RES, SEED)
    return sk, rm, animation_poses(ref, sk), ref.default_camera(sk, width, height), OccupancyConfig(), \
        RenderOptions()
