"""Analytic generators G1-G3; evaluated in float64, stored
float32 [z, y, x] (x fastest).  Each generator is a function of continuous
node-unit positions so ground truth exists at any resolution (2x decode).
Generator parameters come from numpy's default_rng(seed) (harness only)."""
import math

import numpy as np
import torch

SEED = 0x230410516


def _params_g1(seed, k=16):
    r = np.random.default_rng(seed)
    return dict(a=r.uniform(0.5, 1.0, k), c=r.uniform(0.15, 0.85, (k, 3)), s=r.uniform(0.04, 0.12, k))


def _params_g2(seed, m=32):
    r = np.random.default_rng(seed + 2)
    kdir = r.normal(size=(m, 3))
    kdir /= np.linalg.norm(kdir, axis=1, keepdims=True)
    kmag = 2 * math.pi * r.uniform(1.0, 8.0, m)
    return dict(k=kdir * kmag[:, None], phi=r.uniform(0, 2 * math.pi, m))


def _params_g3(seed, waves=256, n=512):
    r = np.random.default_rng(seed + 3)
    kappa = np.exp(r.uniform(0.0, math.log(max(n / 8.0, 2.0)), waves))
    d = r.normal(size=(waves, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    amp = kappa ** -1.4
    amp *= math.sqrt(2.0 / np.sum(amp ** 2))          # unit variance of the sum of cosines
    return dict(k=2 * math.pi * d * kappa[:, None], amp=amp, phi=r.uniform(0, 2 * math.pi, waves))


def evaluate(kind, pos, dims, seed=SEED, tau=0.35):
    """Field value at node-unit positions pos (..., 3) (x, y, z) of a volume with
    `dims` nodes per axis, float64 torch tensor on pos.device."""
    pos = pos.to(torch.float64)
    dims_t = torch.tensor(dims, dtype=torch.float64, device=pos.device)
    p = pos / (dims_t - 1).clamp(min=1)              # domain coordinate in [0,1]^3
    if kind == "g1":
        pr = _params_g1(seed)
        out = torch.zeros(pos.shape[:-1], dtype=torch.float64, device=pos.device)
        for a, c, s in zip(pr["a"], pr["c"], pr["s"]):
            c_t = torch.tensor(c, dtype=torch.float64, device=pos.device)
            out += a * torch.exp(-((p - c_t) ** 2).sum(-1) / (2 * s * s))
        return out
    if kind == "g2":
        pr = _params_g2(seed)
        vox = 1.0 / max(max(dims) - 1, 1)
        w, wf = 1.5 * vox, 2.0 * vox
        lo = torch.zeros(3, dtype=torch.float64, device=pos.device)
        hi = torch.tensor([0.5, 0.2, 0.2], dtype=torch.float64, device=pos.device)
        q = torch.maximum(lo - p, p - hi).clamp(min=0.0)
        d = torch.sqrt((q * q).sum(-1))                 # distance to the hot box
        R = 0.05 + 0.6 * tau ** 0.6
        a = 1.0 / (1.0 + 2.0 * tau)
        e = 1.0 + 1.5 * a * torch.sigmoid(-d / w) + 0.6 * torch.exp(-((d - R) / wf) ** 2)
        k = torch.tensor(pr["k"], dtype=torch.float64, device=pos.device)
        ph = torch.tensor(pr["phi"], dtype=torch.float64, device=pos.device)
        for m in range(k.shape[0]):
            e = e + 0.02 * torch.sin((p * k[m]).sum(-1) + ph[m])
        return e
    if kind == "g3":
        pr = _params_g3(seed, n=max(dims))
        g = torch.zeros(pos.shape[:-1], dtype=torch.float64, device=pos.device)
        k = torch.tensor(pr["k"], dtype=torch.float64, device=pos.device)
        for m in range(k.shape[0]):
            g += float(pr["amp"][m]) * torch.cos((p * k[m]).sum(-1) + float(pr["phi"][m]))
        return torch.exp(1.5 * g - 1.125)
    raise ValueError(kind)


def lattice(dims, device="cpu", z_range=None):
    """Integer node positions (Nz', Ny, Nx, 3) (x, y, z) float64, optionally a z-slab."""
    z0, z1 = (0, dims[2]) if z_range is None else z_range
    zs = torch.arange(z0, z1, dtype=torch.float64, device=device)
    ys = torch.arange(dims[1], dtype=torch.float64, device=device)
    xs = torch.arange(dims[0], dtype=torch.float64, device=device)
    z, y, x = torch.meshgrid(zs, ys, xs, indexing="ij")
    return torch.stack([x, y, z], dim=-1)


def _volume(kind, dims, seed, device, tau=0.35, slab=16):
    out = torch.empty((dims[2], dims[1], dims[0]), dtype=torch.float32, device=device)
    for z0 in range(0, dims[2], slab):
        z1 = min(z0 + slab, dims[2])
        out[z0:z1] = evaluate(kind, lattice(dims, device, (z0, z1)), dims, seed, tau).to(torch.float32)
    return out


def g1_analytic(n=64, seed=SEED, device="cpu"):
    """G1: sum of 16 Gaussian blobs (cfg1)."""
    return _volume("g1", (n, n, n), seed, device)


def g2_energy(n=256, tau=0.35, seed=SEED, device="cpu"):
    """G2: CloverLeaf3D-shaped blast energy field at time tau (cfg2, cfg4)."""
    return _volume("g2", (n, n, n), seed, device, tau)


def g3_density(n=512, seed=SEED, device="cpu"):
    """G3: log-normal cosmology-density-shaped field (cfg3, cfg5)."""
    return _volume("g3", (n, n, n), seed, device)


def linear_field(dims, a=1.0, b=2.0, c=3.0, d=0.0):
    """f = a x + b y + c z + d on the node lattice."""
    z, y, x = np.meshgrid(np.arange(dims[2]), np.arange(dims[1]), np.arange(dims[0]), indexing="ij")
    return (a * x + b * y + c * z + d).astype(np.float32)


def constant_field(dims, value=0.5):
    return np.full((dims[2], dims[1], dims[0]), value, dtype=np.float32)


def taylor_green(pos, dims, t=0.0, amp=1.0, nu=0.05, drift=0.25):
    """G4: Taylor-Green vortex velocity (the NekRS-TGV stand-in of P:L344-346;
    S:L509 u = sin X cos Y cos Z, v = -cos X sin Y cos Z, w = 0) on X = 2 pi
    p / (N - 1) per axis, made time-dependent by viscous decay exp(-2 nu t) and a
    phase drift X -> X - 2 pi drift t.  Velocity in node units per time unit
    (amp = peak speed).  pos (..., 3) float64 torch -> (..., 3)."""
    pos = pos.to(torch.float64)
    dims_t = torch.tensor(dims, dtype=torch.float64, device=pos.device)
    X = 2 * math.pi * pos / (dims_t - 1).clamp(min=1)
    x = X[..., 0] - 2 * math.pi * drift * t
    y, z = X[..., 1], X[..., 2]
    a = amp * math.exp(-2.0 * nu * t)
    u = a * torch.sin(x) * torch.cos(y) * torch.cos(z)
    v = -a * torch.cos(x) * torch.sin(y) * torch.cos(z)
    return torch.stack([u, v, torch.zeros_like(u)], dim=-1)


def taylor_green_volume(n, t=0.0, amp=1.0, device="cpu", **kw):
    """G4 on the n^3 node lattice: float32 [z, y, x, 3] (channels interleaved)."""
    dims = (n, n, n)
    return taylor_green(lattice(dims, device), dims, t, amp, **kw).to(torch.float32)


def random_points(q, dims, seed=SEED):
    """q uniform global node coordinates in [0, N-1]^3, float32 (q, 3)."""
    r = np.random.default_rng(seed + 7)
    return (r.random((q, 3)) * (np.asarray(dims, np.float64) - 1)).astype(np.float32)
