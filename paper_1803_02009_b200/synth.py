"""Seeded synthetic workloads shaped like the paper's laparoscope sequences.

This module is the ONLY code shared by the oracle side (tests) and the CUDA
side (bench / tests).  It holds none of the method's arithmetic: no warp
(Eq. 1), no skinning weights (Eq. 2), no energies, no association, no fusion.
It only synthesises a scene (a deforming height-field surface seen by a moving
pinhole camera) and samples inputs from it:

* model points (positions, analytic normals, colours, fusion weights, stamps)
  of the surface at frame t-1, in world coordinates (mm);
* ED node positions (a regular grid lifted onto the surface) and the node
  neighbour lists N(j) (graph structure, an input of ``mis_set_graph``);
* the observation at frame t: a ray-cast depth map (mm) with Gaussian noise and
  hole discs, an RGB raster, the true world->camera pose and sparse feature
  pairs (model point at t-1 in world coords, its true camera-frame position
  at t plus noise).

Recipe (SURVEY §8(d) "Synthetic inputs"):
laparoscope 40-70 mm from tissue, tissue pushed 2-3 mm at a
random surface point per frame (Table I protocol), respiration
motion, camera motion <= 2 mm / 2 deg per frame,
depth noise sigma 0.1 mm, ~3 % holes (specular highlights).
Seeds: numpy PCG64(1803020090 + 10*cfg_index + frame).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

SEED_BASE = 1803020090


@dataclass(frozen=True)
class SceneConfig:
    name: str
    index: int
    H: int
    W: int
    n_points: int
    m_nodes: int
    k: int
    n_nbr: int
    gn_iters: int
    pcg_iters: int
    n_feat: int
    visible_frac: float
    frames: int = 1


# BASELINE.json "configs"; bracketed values there are
# the survey's proposals and are used as-is.
CONFIGS = {
    "c1": SceneConfig("c1", 1, 64, 80, 5_000, 16, 4, 4, 5, 10, 8, 0.9),
    "c2": SceneConfig("c2", 2, 288, 360, 100_000, 300, 4, 4, 10, 10, 200, 0.9),
    "c3": SceneConfig("c3", 3, 480, 640, 300_000, 1_000, 4, 4, 5, 10, 500, 0.9, frames=100),
    "c4": SceneConfig("c4", 4, 1024, 1280, 2_000_000, 4_000, 4, 4, 5, 10, 1_000, 0.65),
    "c5": SceneConfig("c5", 5, 1024, 1280, 10_000_000, 16_384, 8, 8, 8, 20, 2_000, 0.5),
}

Z0 = 55.0            # mean tissue distance (mm), inside the paper's 40-70 mm
CURV = 300.0         # paraboloid z = Z0 + (x^2+y^2)/CURV
RESP_AMP = 1.5       # respiration amplitude (mm)
RESP_HZ = 0.25       # respiration frequency (Hz)
FPS = 30.0           # PAPER.md:523 (30 fps porcine data)
BUMP_SIGMA = 8.0     # mm
DEPTH_SIGMA = 0.1    # mm
NOISE_CORR_MM = 1.0  # correlation length of the depth noise on the tissue (mm)
WHITE_SIGMA = 0.005  # mm, uncorrelated part
FEAT_SIGMA = 0.2     # mm
HOLE_FRAC = 0.03


def rng_for(cfg: SceneConfig, frame: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + 10 * cfg.index + frame))


def intrinsics(cfg: SceneConfig):
    """Pinhole, fx = fy = 0.714 W (~70 deg horizontal FOV), centre at W/2, H/2."""
    f = float(np.float32(0.714 * cfg.W))   # float32-representable: both sides see the same value
    return dict(fx=f, fy=f, cx=cfg.W / 2.0, cy=cfg.H / 2.0, W=cfg.W, H=cfg.H)


@dataclass
class Surface:
    """Height field z = h(x, y) in world (first camera) coordinates, mm."""
    t_s: float
    bumps: list = field(default_factory=list)   # (bx, by, amp, sigma)

    def h(self, x, y):
        z = Z0 + (x * x + y * y) / CURV + RESP_AMP * math.sin(2 * math.pi * RESP_HZ * self.t_s)
        for bx, by, a, s in self.bumps:
            z = z + a * np.exp(-((x - bx) ** 2 + (y - by) ** 2) / (2 * s * s))
        return z

    def grad(self, x, y):
        hx = 2 * x / CURV
        hy = 2 * y / CURV
        for bx, by, a, s in self.bumps:
            e = a * np.exp(-((x - bx) ** 2 + (y - by) ** 2) / (2 * s * s))
            hx = hx - e * (x - bx) / (s * s)
            hy = hy - e * (y - by) / (s * s)
        return hx, hy

    def h_grad(self, x, y):
        """h and its gradient with one exponential per bump (the ray caster's Newton step)."""
        z = Z0 + (x * x + y * y) / CURV + RESP_AMP * math.sin(2 * math.pi * RESP_HZ * self.t_s)
        hx = 2 * x / CURV
        hy = 2 * y / CURV
        for bx, by, a, s in self.bumps:
            dx, dy = x - bx, y - by
            e = a * np.exp(-(dx * dx + dy * dy) / (2 * s * s))
            z = z + e
            hx = hx - e * dx / (s * s)
            hy = hy - e * dy / (s * s)
        return z, hx, hy

    def normal(self, x, y):
        """Unit normal facing the camera (negative z side)."""
        hx, hy = self.grad(x, y)
        n = np.stack([hx, hy, -np.ones_like(hx)], axis=-1)
        return n / np.linalg.norm(n, axis=-1, keepdims=True)


def rot_xyz(ax, ay, az):
    cx_, sx_ = math.cos(ax), math.sin(ax)
    cy_, sy_ = math.cos(ay), math.sin(ay)
    cz_, sz_ = math.cos(az), math.sin(az)
    rx = np.array([[1, 0, 0], [0, cx_, -sx_], [0, sx_, cx_]])
    ry = np.array([[cy_, 0, sy_], [0, 1, 0], [-sy_, 0, cy_]])
    rz = np.array([[cz_, -sz_, 0], [sz_, cz_, 0], [0, 0, 1]])
    return rz @ ry @ rx


def random_motion(rng, max_mm=2.0, max_deg=2.0):
    """A world->camera pose increment with |t| <= max_mm and angle <= max_deg."""
    ang = np.deg2rad(max_deg) * rng.uniform(-1, 1, 3) / math.sqrt(3)
    t = max_mm * rng.uniform(-1, 1, 3) / math.sqrt(3)
    return rot_xyz(*ang), t


def footprint(cfg: SceneConfig):
    """Half extents (X, Y) of the modelled tissue patch around the optical axis."""
    it = intrinsics(cfg)
    zc = Z0 + 3.0
    e = 1.0 / math.sqrt(cfg.visible_frac)
    X = 0.5 * cfg.W / it["fx"] * zc * e
    Y = 0.5 * cfg.H / it["fy"] * zc * e
    return X, Y


def render_depth(cfg, surf: Surface, R, T, rng, noise=True, holes=True):
    """Ray-cast the height field through a world->camera pose (R, T).

    Returns depth (H, W) float32 in mm (camera-frame z), 0 for holes."""
    it = intrinsics(cfg)
    H, W = cfg.H, cfg.W
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    dc = np.stack([(u - it["cx"]) / it["fx"], (v - it["cy"]) / it["fy"], np.ones_like(u)], -1)
    dw = dc @ R          # R^T d  (row vectors)
    o = -R.T @ T         # camera centre in world
    s = np.full(u.shape, Z0 - o[2])
    for _ in range(30):   # Newton on z(s) - h(x(s), y(s)) = 0, to convergence (quadratic: ~5 steps)
        x = o[0] + s * dw[..., 0]
        y = o[1] + s * dw[..., 1]
        z = o[2] + s * dw[..., 2]
        hz, hx, hy = surf.h_grad(x, y)
        f = z - hz
        fp = dw[..., 2] - (hx * dw[..., 0] + hy * dw[..., 1])
        step = f / fp
        s = s - step
        if np.abs(step).max() < 1e-11:
            break
    # a ray whose Newton iteration has not converged (grazing incidence: f' ~ 0 throws s far away) or
    # that lands behind the camera / beyond 3 Z0 has no valid surface hit: a hole, as in a stereo map
    x = o[0] + s * dw[..., 0]
    y = o[1] + s * dw[..., 1]
    hz, _, _ = surf.h_grad(x, y)
    bad = ~(np.abs(o[2] + s * dw[..., 2] - hz) < 1e-6) | ~(s > 0) | ~(s < 3 * Z0)
    # the camera-frame z of o + s*dw equals s (dc has unit z)
    depth = np.where(bad, 0.0, s)
    if noise:
        # stereo (ELAS-like) depth noise is spatially correlated: a smooth field of
        # std DEPTH_SIGMA (correlation ~NOISE_CORR_MM on the tissue) plus a small
        # white part.  i.i.d. 0.1 mm noise at 0.1-0.2 mm pixels would make
        # central-difference normals ~15-20 deg noisy, failing every 10 deg gate.
        from scipy.ndimage import gaussian_filter
        pix_mm = Z0 / it["fx"]
        sig_px = max(0.5, NOISE_CORR_MM / pix_mm)
        field_ = gaussian_filter(rng.normal(0.0, 1.0, depth.shape), sig_px, mode="reflect")
        field_ *= DEPTH_SIGMA / max(field_.std(), 1e-12)
        depth += field_ + rng.normal(0.0, WHITE_SIGMA, depth.shape)
        depth[bad] = 0.0
    if holes:
        target = HOLE_FRAC * H * W
        r = max(1.5, 0.02 * W)
        n_disc = max(1, int(round(target / (math.pi * r * r))))
        cxs = rng.uniform(0, W, n_disc)
        cys = rng.uniform(0, H, n_disc)
        for a, b in zip(cxs, cys):
            depth[(u - a) ** 2 + (v - b) ** 2 < r * r] = 0.0
    return depth.astype(np.float32)


def texture(x, y):
    """Smooth analytic RGB in [0, 1] as a function of world (x, y)."""
    return np.stack([
        0.5 + 0.4 * np.sin(0.31 * x + 0.7) * np.cos(0.17 * y),
        0.5 + 0.4 * np.sin(0.23 * y + 1.3),
        0.5 + 0.4 * np.cos(0.11 * (x + y)),
    ], -1)


def node_graph(g: np.ndarray, n_nbr: int) -> np.ndarray:
    """N(j): the n_nbr nearest other nodes, ties to the lower id (graph input)."""
    m = g.shape[0]
    nn = min(n_nbr, m - 1)
    out = np.full((m, n_nbr), -1, np.int32)
    g64 = g.astype(np.float64)
    for s in range(0, m, 1024):
        d = ((g64[s:s + 1024, None, :] - g64[None, :, :]) ** 2).sum(-1)
        d[np.arange(d.shape[0]), np.arange(s, s + d.shape[0])] = np.inf
        order = np.argsort(d, axis=1, kind="stable")[:, :nn]
        out[s:s + d.shape[0], :nn] = order
    return out


def sample_model(cfg: SceneConfig, surf_prev: "Surface", rng, frame: int):
    """Model points and ED nodes sampled from the surface at frame-1."""
    X, Y = footprint(cfg)
    # ---- model points: jittered grid over the patch, on the surface at t-1
    n = cfg.n_points
    npx = max(2, int(round(math.sqrt(n * X / Y))))
    npy = max(2, int(math.ceil(n / npx)))
    sx, sy = 2 * X / npx, 2 * Y / npy
    gx, gy = np.meshgrid(-X + sx * (np.arange(npx) + 0.5), -Y + sy * (np.arange(npy) + 0.5))
    px = gx.ravel() + rng.uniform(-0.3, 0.3, gx.size) * sx
    py = gy.ravel() + rng.uniform(-0.3, 0.3, gy.size) * sy
    px, py = px[:n], py[:n]
    pz = surf_prev.h(px, py)
    xyz = np.stack([px, py, pz], -1)
    nrm = surf_prev.normal(px, py)
    rgb = texture(px, py)
    weight = rng.integers(1, 11, n).astype(np.float32)
    stamp = (frame - 1 - rng.integers(0, 6, n)).astype(np.int32)

    # ---- nodes: regular grid over the patch lifted onto the surface at t-1
    m = cfg.m_nodes
    nx = max(1, int(round(math.sqrt(m * X / Y))))
    ny = max(1, int(round(m / nx)))
    ex, ey = 2 * X / nx, 2 * Y / ny
    nxg, nyg = np.meshgrid(-X + ex * (np.arange(nx) + 0.5), -Y + ey * (np.arange(ny) + 0.5))
    gxv = nxg.ravel() + rng.uniform(-0.05, 0.05, nxg.size) * ex   # break exact ties
    gyv = nyg.ravel() + rng.uniform(-0.05, 0.05, nyg.size) * ey
    g = np.stack([gxv, gyv, surf_prev.h(gxv, gyv)], -1)
    nbr = node_graph(g, cfg.n_nbr)

    return dict(xyz=xyz.astype(np.float32), nrm=nrm.astype(np.float32), rgb=rgb.astype(np.float32),
                weight=weight, stamp=stamp, ids=np.arange(n, dtype=np.int64),
                g=g.astype(np.float32), nbr=nbr)


def make_scene(cfg: SceneConfig | str, frame: int = 1, seed_offset: int = 0):
    """Model at frame-1 plus the observation of frame ``frame``.

    Returns a dict of numpy arrays (float32 / int32), all lengths in mm."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = rng_for(cfg, frame + seed_offset)
    X, Y = footprint(cfg)
    t_prev = (frame - 1) / FPS
    t_cur = frame / FPS
    bumps_prev = [(rng.uniform(-X, X) * 0.7, rng.uniform(-Y, Y) * 0.7, rng.uniform(2, 3), BUMP_SIGMA)]
    surf_prev = Surface(t_prev, bumps_prev)
    bumps_cur = bumps_prev + [(rng.uniform(-X, X) * 0.7, rng.uniform(-Y, Y) * 0.7,
                               rng.uniform(2, 3), BUMP_SIGMA)]
    surf_cur = Surface(t_cur, bumps_cur)

    model = sample_model(cfg, surf_prev, rng, frame)
    xyz = model['xyz'].astype(np.float64)

    # ---- observation at frame t through the true pose
    if frame == 1:
        R_prev, T_prev = np.eye(3), np.zeros(3)
    else:
        R_prev, T_prev = rot_xyz(*(0.01 * rng.uniform(-1, 1, 3))), rng.uniform(-1, 1, 3)
    dR, dT = random_motion(rng)
    R = dR @ R_prev
    T = dR @ T_prev + dT
    depth = render_depth(cfg, surf_cur, R, T, rng)
    it = intrinsics(cfg)
    u, v = np.meshgrid(np.arange(cfg.W, dtype=np.float64), np.arange(cfg.H, dtype=np.float64))
    # colour raster: texture at the world point seen by the pixel (approximate: ray at depth)
    dc = np.stack([(u - it["cx"]) / it["fx"] * depth, (v - it["cy"]) / it["fy"] * depth, depth], -1)
    pw = (dc - T) @ R
    rgb_obs = texture(pw[..., 0], pw[..., 1]) + rng.normal(0, 0.01, pw.shape)

    # ---- sparse features: visible model points and their true positions at t
    nf = cfg.n_feat
    cam_prev = xyz @ R.T + T
    inside = (cam_prev[:, 2] > 1) & (np.abs(cam_prev[:, 0] / cam_prev[:, 2]) < 0.4 * cfg.W / it["fx"]) \
        & (np.abs(cam_prev[:, 1] / cam_prev[:, 2]) < 0.4 * cfg.H / it["fy"])
    cand = np.flatnonzero(inside)
    sel = rng.choice(cand, size=min(nf, cand.size), replace=False)
    fsrc = xyz[sel]
    moved = np.stack([fsrc[:, 0], fsrc[:, 1], surf_cur.h(fsrc[:, 0], fsrc[:, 1])], -1)
    fdst = moved @ R.T + T + rng.normal(0, FEAT_SIGMA, moved.shape)

    pose = np.concatenate([R.ravel(), T]).astype(np.float32)
    return dict(
        cfg=cfg, intr=it, **model,
        depth=depth, rgb_obs=rgb_obs.astype(np.float32), pose=pose,
        feat_src=fsrc.astype(np.float32), feat_dst=fdst.astype(np.float32),
        frame=frame,
    )


def make_sequence_frames(cfg: SceneConfig | str, n_frames: int, seed_offset: int = 0):
    """Observations for frames 1..n_frames of a sequence whose model starts at frame 0.

    Each frame adds one 2-3 mm bump and a random camera motion.
    Returns (scene_at_frame_1, [frame dicts with depth, rgb_obs, pose, feat_src, feat_dst])."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = rng_for(cfg, 1000 + seed_offset)
    X, Y = footprint(cfg)
    bumps = [(0.0, 0.0, 2.5, BUMP_SIGMA)]
    base = dict(cfg=cfg, intr=intrinsics(cfg), frame=0, **sample_model(cfg, Surface(0.0, bumps), rng, 0))
    R, T = np.eye(3), np.zeros(3)
    frames = []
    it = intrinsics(cfg)
    for f in range(1, n_frames + 1):
        bumps = bumps + [(rng.uniform(-X, X) * 0.7, rng.uniform(-Y, Y) * 0.7, rng.uniform(2, 3) *
                          (1 if rng.uniform() < 0.5 else -1), BUMP_SIGMA)]
        bumps = bumps[-4:]
        surf = Surface(f / FPS, bumps)
        dR, dT = random_motion(rng)
        R, T = dR @ R, dR @ T + dT
        depth = render_depth(cfg, surf, R, T, rng)
        u, v = np.meshgrid(np.arange(cfg.W, dtype=np.float64), np.arange(cfg.H, dtype=np.float64))
        dc = np.stack([(u - it["cx"]) / it["fx"] * depth, (v - it["cy"]) / it["fy"] * depth, depth], -1)
        pw = (dc - T) @ R
        rgb_obs = texture(pw[..., 0], pw[..., 1])
        frames.append(dict(depth=depth, rgb_obs=rgb_obs.astype(np.float32),
                           pose=np.concatenate([R.ravel(), T]).astype(np.float32), frame=f,
                           feat_src=np.zeros((0, 3), np.float32), feat_dst=np.zeros((0, 3), np.float32)))
    return base, frames
