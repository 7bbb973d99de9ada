"""Training-data sampler for one block ("sampling input coordinates
uniformly within the volume bounding box and computing the corresponding
target values through appropriate interpolation methods utilizing reference
data"; "normalization of both input coordinates and output values to
the range [0,1]"), made concrete by S:L39-47, S:L66-92 and
DESIGN.md readings R5-R9.

Volumes are numpy arrays indexed [z, y, x] (x-fastest in memory); a node
(ix, iy, iz) sits at integer position p = (ix, iy, iz).  A block has core
origin o and n cells per axis; its normalized coordinate is x = (p - o) / n
(cell-span convention, R5), so adjacent blocks share the face plane o + n.
"""
import numpy as np

from . import philox

FACE_NAMES = ("-x", "+x", "-y", "+y", "-z", "+z")


class Block:
    """origin (3,) nodes, n (3,) cells per axis, global_dims (3,) nodes; all (x, y, z).
    mesh: None (uniform) or three strictly increasing float64 arrays of the
    global node coordinates per axis (rectilinear; R36)."""

    def __init__(self, origin, n, global_dims, mesh=None):
        self.origin = np.asarray(origin, dtype=np.int64)
        self.n = np.asarray(n, dtype=np.int64)
        self.global_dims = np.asarray(global_dims, dtype=np.int64)
        self.mesh = None if mesh is None else tuple(np.asarray(m, np.float64) for m in mesh)

    def physical_box(self):
        """(P_lo, P_hi) of a rectilinear block: the coordinates of nodes o and
        min(o + n, N - 1) per axis (R36)."""
        lo = np.array([self.mesh[d][self.origin[d]] for d in range(3)])
        hi = np.array([self.mesh[d][min(self.origin[d] + self.n[d], self.global_dims[d] - 1)] for d in range(3)])
        return lo, hi

    @property
    def grid(self):
        """Blocks per axis B_d = ceil(N_d / n_d) (divisible decomposition)."""
        return (self.global_dims + self.n - 1) // self.n

    @property
    def block_id(self):
        """Linear block index, x fastest: (o_z/n_z * B_y + o_y/n_y) * B_x + o_x/n_x."""
        c = self.origin // self.n
        g = self.grid
        return int((c[2] * g[1] + c[1]) * g[0] + c[0])

    def interior_faces(self):
        """Faces shared with a neighbouring block, ordered -x,+x,-y,+y,-z,+z
        (domain-exterior faces excluded)."""
        out = []
        for d in range(3):
            if self.origin[d] > 0:
                out.append(2 * d)
            if self.origin[d] + self.n[d] < self.global_dims[d]:
                out.append(2 * d + 1)
        return out


def decompose(global_dims, n, mesh=None):
    """All blocks of a volume, in block_id order."""
    gd = np.asarray(global_dims, np.int64)
    n = np.asarray(n, np.int64)
    g = (gd + n - 1) // n
    return [Block((bx * n[0], by * n[1], bz * n[2]), n, gd, mesh)
            for bz in range(g[2]) for by in range(g[1]) for bx in range(g[0])]


def uniform_samples(seed, step, block_id, count):
    """x_i ~ U[0,1)^3, i < count: (u0,u1,u2,.) = Philox4x32-10(key(seed, 1),
    ctr = (i, step, block_id, 0)); x_d = (u_d >> 8) 2^-24 (R8).  float32 (count, 3)."""
    i = np.arange(count, dtype=np.uint64)
    key = philox.stream_key(seed, 1)
    u = philox.philox4x32_10((i, np.full_like(i, step), np.full_like(i, block_id), np.zeros_like(i)), key)
    return np.stack([philox.u01(u[0]), philox.u01(u[1]), philox.u01(u[2])], axis=1)


def boundary_samples(seed, step, block, count):
    """Samples exactly on the block's interior faces (P:L198-202 X_Bound; R9):
    Philox(key(seed, 2), ctr = (j, step, block_id, 0)); face =
    interior_faces[((u0 >> 8) * n_faces) >> 24]; the normal coordinate is 0
    (minus face) or 1 (plus face); the two in-face coordinates, in axis order,
    are u01(u1), u01(u2).  Returns float32 (count, 3); empty if no interior face."""
    faces = block.interior_faces()
    if count <= 0 or not faces:
        return np.zeros((0, 3), dtype=np.float32)
    j = np.arange(count, dtype=np.uint64)
    key = philox.stream_key(seed, 2)
    u = philox.philox4x32_10((j, np.full_like(j, step), np.full_like(j, block.block_id), np.zeros_like(j)), key)
    sel = ((u[0].astype(np.uint64) >> np.uint64(8)) * np.uint64(len(faces))) >> np.uint64(24)
    face = np.asarray(faces, dtype=np.int64)[sel.astype(np.int64)]
    a = philox.u01(u[1])
    b = philox.u01(u[2])
    x = np.empty((count, 3), dtype=np.float32)
    for fcode in range(6):
        m = face == fcode
        if not np.any(m):
            continue
        d = fcode // 2
        others = [e for e in range(3) if e != d]
        x[m, d] = np.float32(fcode % 2)
        x[m, others[0]] = a[m]
        x[m, others[1]] = b[m]
    return x


def trilinear(volume, r):
    """Trilinear interpolation of volume[z, y, x] (scalar) or volume[z, y, x, c]
    (D channels, interleaved) at node-unit positions r (n,3) (x, y, z), per
    channel, with clamp-to-edge at the global faces (R5).  Float64;
    returns (n,) or (n, D)."""
    vol = np.asarray(volume)
    dims = np.array([vol.shape[2], vol.shape[1], vol.shape[0]], dtype=np.int64)
    r = np.clip(np.asarray(r, np.float64), 0.0, (dims - 1).astype(np.float64))
    i0 = np.floor(r).astype(np.int64)
    f = r - i0
    i1 = np.minimum(i0 + 1, dims - 1)
    out = np.zeros((r.shape[0],) + vol.shape[3:], dtype=np.float64)
    for c in range(8):
        b = [(c >> d) & 1 for d in range(3)]
        ix = i1[:, 0] if b[0] else i0[:, 0]
        iy = i1[:, 1] if b[1] else i0[:, 1]
        iz = i1[:, 2] if b[2] else i0[:, 2]
        w = np.ones(r.shape[0])
        for d in range(3):
            w = w * (f[:, d] if b[d] else 1.0 - f[:, d])
        out += w.reshape((-1,) + (1,) * (vol.ndim - 3)) * vol[iz, iy, ix].astype(np.float64)
    return out


def normalize_values(v, vmin, vmax):
    """t = (v - vmin) / (vmax - vmin) with the shared global range (
    S:L66-74), per channel for vector fields (vmin, vmax of shape (D,)
    "normalized per-channel with a shared global range per channel").  A
    constant channel (vmax == vmin) gives t = 0.
    Returns (t, constant_flag), the flag set when every channel is constant."""
    v = np.asarray(v, np.float64)
    lo = np.asarray(vmin, np.float64)
    hi = np.asarray(vmax, np.float64)
    span = hi - lo
    const = span == 0.0
    t = (v - lo) / np.where(const, 1.0, span)
    t = np.where(const, 0.0, t)
    return t, bool(np.all(const))


def physical_to_index(coords, P):
    """Continuous node index of physical coordinates P on one rectilinear axis:
    r = i + (P - X_i) / (X_{i+1} - X_i), X_i <= P <= X_{i+1}, i clipped to the
    mesh's cells, so trilinear in r is trilinear in the physical cell (R36)."""
    X = np.asarray(coords, np.float64)
    P = np.asarray(P, np.float64)
    i = np.clip(np.searchsorted(X, P, side="right") - 1, 0, X.size - 2)
    return i + (P - X[i]) / (X[i + 1] - X[i])


def index_to_physical(coords, r):
    """The mesh's piecewise-linear map from continuous node index to coordinate."""
    X = np.asarray(coords, np.float64)
    r = np.asarray(r, np.float64)
    i = np.clip(np.floor(r).astype(np.int64), 0, X.size - 2)
    return X[i] + (r - i) * (X[i + 1] - X[i])


def sample_positions(block, x):
    """Node-index positions r (n, 3) of block-normalized samples x: r = o + x n on a
    uniform mesh (R5); on a rectilinear mesh the physical point P = P_lo + x (P_hi -
    P_lo) of the block's box mapped to its continuous index (R36)."""
    x = np.asarray(x, np.float64)
    if block.mesh is None:
        return block.origin[None, :].astype(np.float64) + x * block.n[None, :].astype(np.float64)
    lo, hi = block.physical_box()
    P = lo[None, :] + x * (hi - lo)[None, :]
    return np.stack([physical_to_index(block.mesh[d], P[:, d]) for d in range(3)], axis=1)


def targets(volume, block, x, vmin, vmax):
    """Reference targets at block-normalized x: trilinear at the sample's node
    position (R5 / R36), normalized with the global range (R7)."""
    return normalize_values(trilinear(volume, sample_positions(block, x)), vmin, vmax)


def value_range(volumes):
    """Global (vmin, vmax) over all core nodes of all partitions, as the range
    all-reduce computes it ("normalized using the same maximum and
    minimum values"; R7).  Scalars for scalar fields; per-channel
    arrays (D,) for vector fields volume[z, y, x, c]."""
    if np.asarray(volumes[0]).ndim == 4:
        lo = np.min([np.min(v, axis=(0, 1, 2)) for v in volumes], axis=0).astype(np.float64)
        hi = np.max([np.max(v, axis=(0, 1, 2)) for v in volumes], axis=0).astype(np.float64)
        return lo, hi
    lo = min(float(np.min(v)) for v in volumes)
    hi = max(float(np.max(v)) for v in volumes)
    return lo, hi


def probe_lattice(m=32):
    """Cell-centred probe positions x = (j + 0.5)/m per axis, x fastest."""
    g = (np.arange(m, dtype=np.float64) + 0.5) / m
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    return np.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], axis=1).astype(np.float32)


def psnr(pred, ref):
    """PSNR = -10 log10(MSE), peak 1 on [0,1]-normalized values, capped at
    200 dB (R18)."""
    mse = float(np.mean((np.asarray(pred, np.float64) - np.asarray(ref, np.float64)) ** 2))
    return psnr_from_mse(mse)


def psnr_from_mse(mse):
    if mse <= 0.0:
        return 200.0
    return min(200.0, -10.0 * np.log10(mse))
