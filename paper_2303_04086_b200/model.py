"""Host-side render state, attribute-compatible with the reference's types.

The reference's objects (radfarm.core.Camera, radfarm.lightfield.LightFieldAsset,
...) can be passed to every function of this package unchanged: only their
attributes are read.  These classes exist so the package runs where the
reference is absent (the GPU box) and are field-for-field the same surface:

  Aabb, Camera, Frame                 core.py:62-159
  MarchParams, ModelWiring,
  RenderCounters, LightFieldAsset     lightfield.py:59-126, 217-248
  CubeAtlas                           atlas.py:25-51
  PshTable                            encoding.py:109-140
  HashGridEncoder                     encoding.py:405-433
  Mlp                                 neural.py:29-71
  RayRange, Tile                      renderer.py:16-53
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import errors

DEPTH_MISS = np.float32(np.inf)
PRIMES_H0 = np.array([1, 2654435761, 805459861], dtype=np.uint64)
PRIMES_H1 = np.array([73856093, 19349663, 83492791], dtype=np.uint64)


def _vec3(v) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (3,):
        raise errors.DomainError(f"expected 3-vector, got shape {a.shape}")
    return a


@dataclass(frozen=True)
class Aabb:
    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "min", _vec3(self.min))
        object.__setattr__(self, "max", _vec3(self.max))
        if not np.all(self.min <= self.max):
            raise errors.DomainError("Aabb requires min <= max componentwise")

    @property
    def diagonal(self) -> float:
        return float(np.linalg.norm(self.max - self.min))

    def corners(self) -> np.ndarray:
        bits = (np.arange(8)[:, None] >> np.arange(3)[None, :]) & 1
        return np.where(bits.astype(bool), self.max, self.min)


UNIT_BOX = Aabb(min=(0.0, 0.0, 0.0), max=(1.0, 1.0, 1.0))


@dataclass(frozen=True)
class Camera:
    pose: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        pose = np.asarray(self.pose, dtype=np.float64)
        if pose.shape != (4, 4):
            raise errors.DomainError("camera pose must be 4x4")
        rot = pose[:3, :3]
        if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-5):
            raise errors.DomainError("camera pose rotation block must be orthonormal")
        if not (self.fx > 0 and self.fy > 0):
            raise errors.DomainError("focal lengths must be positive")
        if self.width < 1 or self.height < 1:
            raise errors.DomainError("image must be at least 1x1")
        object.__setattr__(self, "pose", pose)

    @property
    def position(self) -> np.ndarray:
        return self.pose[:3, 3]

    @property
    def rotation(self) -> np.ndarray:
        return self.pose[:3, :3]


@dataclass
class Frame:
    width: int
    height: int
    rgba: np.ndarray
    depth: np.ndarray

    @classmethod
    def empty(cls, width: int, height: int) -> "Frame":
        return cls(width, height, np.zeros((height, width, 4), np.float32),
                   np.full((height, width), DEPTH_MISS, np.float32))


# protocol.py:36-37 frame encodings
ENC_RAW = 0
ENC_DEFLATE = 1


@dataclass
class FrameData:
    """protocol.FrameData (protocol.py:71-80): an encoded frame message."""
    pose_seq: int
    frame_index: int
    encoding: int
    width: int
    height: int
    depth_far: float
    rgba: bytes
    depth: bytes


@dataclass
class MarchParams:
    step: float
    t_stop: float = 1e-4
    alpha_floor: float = 1e-4


@dataclass(frozen=True)
class ModelWiring:
    use_hit_point: bool = True
    use_opacity: bool = True
    refine_opacity: bool = True
    use_tint: bool = True
    use_diffuse_color: bool = True


@dataclass
class RenderCounters:
    fs_evals: int = 0
    fd_evals: int = 0
    hit_pixels: int = 0
    march_samples: int = 0

    def merge(self, other) -> None:
        self.fs_evals += other.fs_evals
        self.fd_evals += other.fd_evals
        self.hit_pixels += other.hit_pixels
        self.march_samples += other.march_samples


@dataclass
class CubeAtlas:
    base_resolution: int
    cube_resolution: int
    channels: int
    index: np.ndarray
    cubes: np.ndarray

    @property
    def cube_count(self) -> int:
        return len(self.cubes)


@dataclass
class PshTable:
    resolution: int
    table_size: int
    offset_size: int
    offsets: np.ndarray
    report: object = None
    primes_h0: np.ndarray = field(default_factory=lambda: PRIMES_H0.copy())
    primes_h1: np.ndarray = field(default_factory=lambda: PRIMES_H1.copy())


@dataclass
class HashGridEncoder:
    levels: int
    base_resolution: int
    growth: float
    table_size: int
    features_per_level: int

    def __post_init__(self):
        # encoding.py:415-424: same float expression, same integer results
        self.resolutions = [max(2, int(math.floor(self.base_resolution * self.growth ** l)))
                            for l in range(self.levels)]
        self.dense = [(n + 1) ** 3 <= self.table_size for n in self.resolutions]
        self.row_counts = [(n + 1) ** 3 if d else self.table_size
                           for n, d in zip(self.resolutions, self.dense)]

    @property
    def output_dim(self) -> int:
        return self.levels * self.features_per_level


@dataclass
class Mlp:
    weights: list
    biases: list
    heads: tuple

    @property
    def input_dim(self) -> int:
        return self.weights[0].shape[1]

    def parameters(self) -> list:
        """neural.Mlp.parameters (neural.py:65-66): weights then biases."""
        return list(self.weights) + list(self.biases)


@dataclass
class LightFieldAsset:
    density_atlas: CubeAtlas | None
    psh: PshTable | None
    psh_features: np.ndarray | None
    diffuse_encoder: HashGridEncoder | None
    diffuse_features: list | None
    specular_mlp: Mlp | None
    diffuse_mlp: Mlp | None
    march: MarchParams
    proxy: Aabb = field(default_factory=lambda: UNIT_BOX)
    object_to_world: np.ndarray = field(default_factory=lambda: np.eye(4))
    diffuse_atlas: CubeAtlas | None = None
    wiring: ModelWiring = field(default_factory=ModelWiring)
    analytic_density: object = None
    analytic_color: object = None
    name: str = "asset"
    # optional triangle-mesh proxy (vertices (n,3) f64, triangles (m,3) int32),
    # object space inside `proxy`; the march starts at its first hit.  Not in
    # the reference (BASELINE config 2).
    proxy_mesh: tuple | None = None


@dataclass(frozen=True)
class RayRange:
    camera: Camera
    x0: int
    y0: int
    x1: int
    y1: int
    asset_id: str = "asset"

    def __post_init__(self):
        if not (0 <= self.x0 < self.x1 <= self.camera.width):
            raise errors.DomainError("ray range x bounds outside frame")
        if not (0 <= self.y0 < self.y1 <= self.camera.height):
            raise errors.DomainError("ray range y bounds outside frame")

    @property
    def pixel_count(self) -> int:
        return (self.x1 - self.x0) * (self.y1 - self.y0)


@dataclass
class Tile:
    x0: int
    y0: int
    rgba: np.ndarray
    depth: np.ndarray

    @property
    def width(self) -> int:
        return self.rgba.shape[1]

    @property
    def height(self) -> int:
        return self.rgba.shape[0]


def uniform_scale_of(matrix) -> float:
    """Uniform scale of a rigid + uniform-scale 4x4 (core.py:273-286)."""
    m = np.asarray(matrix, dtype=np.float64)
    if m.shape != (4, 4):
        raise errors.DomainError("transform must be 4x4")
    lin = m[:3, :3]
    norms = np.linalg.norm(lin, axis=0)
    s = float(norms.mean())
    if s <= 0 or not np.allclose(norms, s, rtol=1e-5):
        raise errors.DomainError("transform must have uniform positive scale")
    rot = lin / s
    if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-5):
        raise errors.DomainError("transform must be rigid + uniform scale")
    return s


def look_at(eye, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """Camera-to-world pose looking from eye to target along -z (core.py:307-323)."""
    eye = _vec3(eye)
    fwd = _vec3(target) - eye
    fwd = fwd / np.linalg.norm(fwd)
    up = _vec3(up)
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-8:
        right = np.cross(fwd, np.array([1.0, 0.0, 0.0]))
    right = right / np.linalg.norm(right)
    true_up = np.cross(right, fwd)
    pose = np.eye(4)
    pose[:3, 0] = right
    pose[:3, 1] = true_up
    pose[:3, 2] = -fwd
    pose[:3, 3] = eye
    return pose


def orbit_camera(azimuth, elevation, radius=2.0, size=64, fov_deg=60.0, target=(0.5, 0.5, 0.5),
                 width=None, height=None) -> Camera:
    """Orbit camera of scenes.py:288-306; ``width``/``height`` allow the
    non-square BASELINE frames (cx = W/2, cy = H/2, fx = fy from the width)."""
    target = np.asarray(target, dtype=np.float64)
    ce, se = math.cos(elevation), math.sin(elevation)
    eye = target + radius * np.array([ce * math.cos(azimuth), ce * math.sin(azimuth), se])
    w = size if width is None else width
    h = size if height is None else height
    fx = w / (2.0 * math.tan(math.radians(fov_deg) / 2.0))
    return Camera(pose=look_at(eye, target, (0.0, 0.0, 1.0)), fx=fx, fy=fx, cx=w / 2, cy=h / 2,
                  width=w, height=h)
