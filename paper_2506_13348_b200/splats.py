"""Camera model and renderer constants (mirrors texsplat.splats).

Reference: /root/reference/pkg/src/texsplat/splats.py:25-140. The camera is a
host-side value object; render calls pass it to libtsb as a tsb_camera.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DENOM_EPS = 1e-9            # splats.py:25
ALPHA_CUTOFF = 1.0 / 255.0  # splats.py:28
SUPPORT_SIGMA = 3.0         # splats.py:31


@dataclass
class Camera:
    """Pinhole camera, view x-right / y-down / z-forward (splats.py:45-78).

    Pixel (px, py) covers camera-plane coordinates
    x = (px + 0.5 - cx) / fx, y = (py + 0.5 - cy) / fy at its centre.
    """

    world_to_view: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.01
    far: float = 100.0

    def __post_init__(self):
        self.world_to_view = np.asarray(self.world_to_view, dtype=np.float64)
        if self.world_to_view.shape != (4, 4):
            raise ValueError("world_to_view must be 4x4")
        R = self.world_to_view[:3, :3]
        if not np.allclose(R @ R.T, np.eye(3), atol=1e-6):
            raise ValueError("world_to_view rotation block is not orthonormal")
        if not np.allclose(self.world_to_view[3], [0.0, 0.0, 0.0, 1.0], atol=1e-9):
            raise ValueError("world_to_view last row must be (0,0,0,1)")
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("image size must be positive")
        if not (0.0 < self.near < self.far):
            raise ValueError("need 0 < near < far")

    @staticmethod
    def look_at(eye, target, up=(0.0, 1.0, 0.0), *, fov_x_deg=60.0, width=256,
                height=256, near=0.01, far=100.0) -> "Camera":
        eye = np.asarray(eye, dtype=np.float64)
        target = np.asarray(target, dtype=np.float64)
        fwd = target - eye
        n = np.linalg.norm(fwd)
        if n < 1e-12:
            raise ValueError("eye and target coincide")
        fwd = fwd / n
        right = np.cross(fwd, np.asarray(up, dtype=np.float64))
        rn = np.linalg.norm(right)
        if rn < 1e-12:
            raise ValueError("up is parallel to the view direction")
        right = right / rn
        down = np.cross(fwd, right)
        R = np.stack([right, down, fwd])
        w2v = np.eye(4)
        w2v[:3, :3] = R
        w2v[:3, 3] = -R @ eye
        fx = 0.5 * width / np.tan(0.5 * np.radians(fov_x_deg))
        return Camera(w2v, fx=fx, fy=fx, cx=0.5 * width, cy=0.5 * height, width=width,
                      height=height, near=near, far=far)

    @property
    def rotation(self) -> np.ndarray:
        return self.world_to_view[:3, :3]

    @property
    def center(self) -> np.ndarray:
        R = self.world_to_view[:3, :3]
        return -R.T @ self.world_to_view[:3, 3]

    def pixel_plane_coords(self):
        xs = (np.arange(self.width, dtype=np.float64) + 0.5 - self.cx) / self.fx
        ys = (np.arange(self.height, dtype=np.float64) + 0.5 - self.cy) / self.fy
        return xs, ys

    def ray_dirs_world(self, x, y) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        d_view = np.stack(np.broadcast_arrays(x, y, np.ones_like(x + y)), axis=-1)
        d_world = d_view @ self.rotation
        return d_world / np.linalg.norm(d_world, axis=-1, keepdims=True)

    def crop(self, x0: int, y0: int, w: int, h: int) -> "Camera":
        """Window (x0, y0, w, h) of this camera; its pixels are identical to
        the same pixels of the full frame."""
        return Camera(self.world_to_view.copy(), fx=self.fx, fy=self.fy, cx=self.cx - x0,
                      cy=self.cy - y0, width=w, height=h, near=self.near, far=self.far)
