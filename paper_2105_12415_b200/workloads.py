"""Seeded synthetic triangle-pair workloads (BASELINE.json configs 0-4).

No dataset ships with the reference: its tests draw pairs from seeded
generators (RT/conftest.py:14-22, RT/test_acceptance.py:32-66), so every
config here is a seeded generator with the shapes and distributions
BASELINE.json names.

Random pairs (cfg0 / cfg1 / cfg4) are prefix-consistent: pair i lives in
chunk ``i // 4096`` which uses ``np.random.default_rng([seed, chunk])``, so
any contiguous range (a shard) can be generated independently and cfg0 is
exactly the first chunk of cfg1.  Draw order per chunk:
A ~ U[0,1]^(4096,3,3); q ~ N(0,1)^(4096,4) normalised (the
``RigidMotion.random_rotation`` construction, RK/geometry.py:156-160 and
its matrix RK/geometry.py:162-171); u ~ N(0,1)^(4096,3) normalised;
s ~ U[lo,hi]^4096.  B = R(q) (A - c_A) + c_A + s u, c_A = centroid of A.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 4096

# (n, seed, sep_lo, sep_hi) of the random-pair configs
CFG0 = dict(n=4096, seed=0, sep=(-0.1, 0.5))
CFG1 = dict(n=1 << 24, seed=0, sep=(-0.1, 0.5))
CFG4 = dict(n=1 << 28, seed=0, sep=(-0.05, 0.2))


def rotation_matrices(q: np.ndarray) -> np.ndarray:
    """(m, 4) unit quaternions (w, x, y, z) -> (m, 3, 3), RK/geometry.py:162-171."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((q.shape[0], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _chunk(seed: int, k: int, sep) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng([seed, k])
    A = rng.random((CHUNK, 3, 3))
    q = rng.normal(size=(CHUNK, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    u = rng.normal(size=(CHUNK, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    s = rng.uniform(sep[0], sep[1], size=CHUNK)
    c = A.mean(axis=1, keepdims=True)
    return A, rotate_about(A, c, rotation_matrices(q), s[:, None] * u)


def rotate_about(A: np.ndarray, c: np.ndarray, R: np.ndarray, t: np.ndarray) -> np.ndarray:
    """R (A - c) + c + t per pair: A (m,3,3), c (m,1,3), R (m,3,3), t (m,3)."""
    X = A - c
    Rt = R[:, None, :, :]
    B = X[:, :, None, 0] * Rt[..., 0] + X[:, :, None, 1] * Rt[..., 1] + X[:, :, None, 2] * Rt[..., 2]
    return B + c + t[:, None, :]


def random_pairs(n: int, seed: int = 0, sep=(-0.1, 0.5), start: int = 0,
                 dtype=np.float64, threads: int = 8, out: tuple | None = None):
    """Pairs [start, start + n) of the chunked generator as (A, B) (n, 3, 3).

    ``out`` may supply preallocated (A, B) arrays (e.g. pinned host memory).
    """
    if out is None:
        A = np.empty((n, 3, 3), dtype)
        B = np.empty((n, 3, 3), dtype)
    else:
        A, B = out
    if n == 0:
        return A, B
    k0 = start // CHUNK
    k1 = (start + n - 1) // CHUNK

    def work(k):
        a, b = _chunk(seed, k, sep)
        lo = max(start, k * CHUNK)
        hi = min(start + n, (k + 1) * CHUNK)
        A[lo - start:hi - start] = a[lo - k * CHUNK:hi - k * CHUNK]
        B[lo - start:hi - start] = b[lo - k * CHUNK:hi - k * CHUNK]

    ks = range(k0, k1 + 1)
    if threads > 1 and len(ks) > 4:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, ks))
    else:
        for k in ks:
            work(k)
    return A, B


def _mp_worker(args):
    name, shape, dtype, seed, sep, start, lo, hi = args
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(name=name)
    try:
        buf = np.ndarray(shape, dtype=dtype, buffer=shm.buf)
        A, B = random_pairs(hi - lo, seed=seed, sep=sep, start=start + lo, dtype=dtype, threads=1)
        buf[0, lo:hi] = A
        buf[1, lo:hi] = B
    finally:
        shm.close()


def random_pairs_mp(n: int, seed: int = 0, sep=(-0.1, 0.5), start: int = 0, dtype=np.float64,
                    processes: int | None = None):
    """random_pairs for large n on all host cores (process pool + shared memory);
    bit-identical to random_pairs (same per-chunk streams)."""
    import multiprocessing as mp
    import os
    from multiprocessing import shared_memory
    processes = processes or len(os.sched_getaffinity(0))
    if processes <= 1 or n < 64 * CHUNK:
        return random_pairs(n, seed=seed, sep=sep, start=start, dtype=dtype)
    shape = (2, n, 3, 3)
    shm = shared_memory.SharedMemory(create=True, size=int(np.prod(shape)) * np.dtype(dtype).itemsize)
    try:
        # split on chunk boundaries of the absolute index so every chunk is generated once
        edges = sorted({0, n} | {min(n, max(0, k * CHUNK - start)) for k in
                                 range(start // CHUNK, (start + n) // CHUNK + 1, max(1, (n // CHUNK) // (4 * processes)))})
        jobs = [(shm.name, shape, np.dtype(dtype).str, seed, sep, start, lo, hi) for lo, hi in zip(edges, edges[1:]) if hi > lo]
        with mp.get_context("fork").Pool(processes) as pool:
            pool.map(_mp_worker, jobs)
        buf = np.ndarray(shape, dtype=dtype, buffer=shm.buf)
        A = buf[0].copy()
        B = buf[1].copy()
    finally:
        shm.close()
        shm.unlink()
    return A, B


def to_soa(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """(n,3,3) x 2 -> planar [18][n]: planes 0-8 are A's v0x..v2z, 9-17 B's."""
    n = A.shape[0]
    out = np.empty((18, n), A.dtype)
    out[:9] = A.reshape(n, 9).T
    out[9:] = B.reshape(n, 9).T
    return out


# ---------------------------------------------------------------------------
# cfg3: adversarial robustness classes (near-parallel, edge-edge, slivers,
# exactly touching), 4 x n_per pairs, concatenated in that order.
# ---------------------------------------------------------------------------

def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _axis_rotation(axis: np.ndarray, angle: np.ndarray) -> np.ndarray:
    half = 0.5 * angle
    q = np.concatenate([np.cos(half)[:, None], np.sin(half)[:, None] * axis], axis=1)
    return rotation_matrices(q)


def near_parallel(rng, m):
    """B = A tilted by < 1e-3 rad about an in-plane axis, lifted by U[0, 0.05]
    along A's normal, and shifted in-plane by up to 0.3."""
    A = rng.random((m, 3, 3))
    c = A.mean(axis=1, keepdims=True)
    nrm = _unit(np.cross(A[:, 1] - A[:, 0], A[:, 2] - A[:, 0]))
    e = _unit(A[:, 1] - A[:, 0])
    f = np.cross(nrm, e)
    phi = rng.uniform(0, 2 * np.pi, m)
    axis = np.cos(phi)[:, None] * e + np.sin(phi)[:, None] * f
    R = _axis_rotation(axis, rng.uniform(0, 1e-3, m))
    lift = rng.uniform(0, 0.05, m)
    shift = rng.uniform(-0.3, 0.3, (m, 2))
    t = lift[:, None] * nrm + shift[:, :1] * e + shift[:, 1:] * f
    return A, rotate_about(A, c, R, t)


def edge_edge(rng, m):
    """A's edge v0-v1 and B's edge w0-w1 cross skew, offset U[0, 0.05] along
    their common normal; both third vertices lie away from the gap."""
    A = rng.random((m, 3, 3))
    da = _unit(A[:, 1] - A[:, 0])
    ma = 0.5 * (A[:, 0] + A[:, 1])
    db = _unit(rng.normal(size=(m, 3)))
    nrm = _unit(np.cross(da, db))
    # keep A's third vertex on the -nrm side
    side = np.einsum("ij,ij->i", A[:, 2] - ma, nrm)
    flip = side > 0
    nrm[flip] *= -1
    h = rng.uniform(0, 0.05, m)
    half = rng.uniform(0.2, 0.6, m)
    mb = ma + h[:, None] * nrm
    B = np.empty_like(A)
    B[:, 0] = mb - half[:, None] * db
    B[:, 1] = mb + half[:, None] * db
    B[:, 2] = mb + rng.uniform(0.2, 0.8, m)[:, None] * nrm + rng.uniform(-0.3, 0.3, (m, 1)) * np.cross(nrm, db)
    # push A's third vertex further to the -nrm side
    A[:, 2] = A[:, 2] - rng.uniform(0.05, 0.3, m)[:, None] * nrm
    return A, B


def slivers(rng, m):
    """A is a sliver of aspect ratio 10^U(4,5); B a random triangle near it."""
    L = rng.uniform(0.5, 1.0, m)
    d = _unit(rng.normal(size=(m, 3)))
    p = _unit(np.cross(d, _unit(rng.normal(size=(m, 3)))))
    aspect = 10.0 ** rng.uniform(4, 5, m)
    v0 = rng.random((m, 3))
    A = np.empty((m, 3, 3))
    A[:, 0] = v0
    A[:, 1] = v0 + L[:, None] * d
    A[:, 2] = v0 + (rng.uniform(0.2, 0.8, m) * L)[:, None] * d + (L / aspect)[:, None] * p
    B = rng.random((m, 3, 3)) * 0.5 + A.mean(axis=1, keepdims=True) - 0.25 + \
        (rng.uniform(-0.05, 0.3, m)[:, None] * _unit(rng.normal(size=(m, 3))))[:, None, :]
    return A, B


def touching(rng, m):
    """Exactly touching vertex-face pairs on a dyadic grid: B's v0 is a dyadic
    point of A's face and B lies in A's closed positive half-space, so the
    exact distance is 0 and every coordinate is exactly representable."""
    A = rng.integers(0, 65, (m, 3, 3)).astype(np.float64) / 64.0
    e1 = A[:, 1] - A[:, 0]
    e2 = A[:, 2] - A[:, 0]
    nrm = np.cross(e1, e2) * 64.0 * 64.0  # integer-valued normal
    bad = np.einsum("ij,ij->i", nrm, nrm) == 0
    A[bad, 2] += np.array([0.0, 0.0, 0.5])
    e2 = A[:, 2] - A[:, 0]
    nrm = np.cross(e1, e2) * 64.0 * 64.0
    a = rng.integers(0, 9, m) / 16.0
    b = rng.integers(0, 9, m) / 16.0
    over = a + b > 1
    a[over], b[over] = 1 - a[over], 1 - b[over]
    B = np.empty_like(A)
    B[:, 0] = A[:, 0] + a[:, None] * e1 + b[:, None] * e2
    scale = 1.0 / np.maximum(np.abs(nrm).max(axis=1), 1.0)
    scale = 2.0 ** np.floor(np.log2(scale))[:, None]  # dyadic
    # B's other vertices: a lift along A's normal plus an in-plane step along
    # A's edge e1 (for v1) or e2 (for v2) -- independent directions, so B is
    # never degenerate, and exactly in the closed positive half-space
    for k, e in ((1, e1), (2, e2)):
        step = rng.integers(1, 5, m)[:, None] / 16.0 * rng.choice([-1.0, 1.0], (m, 1))
        lift = rng.integers(1, 9, m)[:, None] * scale * nrm * 4.0
        B[:, k] = B[:, 0] + step * e + lift
    return A, B


CFG3_CLASSES = ("near_parallel", "edge_edge", "slivers", "touching")


def adversarial_pairs(n_per: int, seed: int = 3):
    """cfg3: the four classes of n_per pairs each, in CFG3_CLASSES order."""
    As, Bs = [], []
    for k, fn in enumerate((near_parallel, edge_edge, slivers, touching)):
        rng = np.random.default_rng([seed, k])
        a, b = fn(rng, n_per)
        As.append(a)
        Bs.append(b)
    return np.concatenate(As), np.concatenate(Bs)


# ---------------------------------------------------------------------------
# Counter-based generator of the same cfg0 distribution (device: the C-ABI
# tc_random_pairs_soa_f64; this numpy mirror checks it).  Pair i draws nine
# Philox4x32-10 blocks with counter (i_lo, i_hi, call, 0) and key
# (seed_lo, seed_hi ^ 0x5EED): 18 uniforms = A (9), s (1), four Box-Muller
# pairs -> q (4), u (3).  Used for the 2^28-pair cfg4 runs, whose host numpy
# generation would take minutes.
# ---------------------------------------------------------------------------
_PH_M0, _PH_M1, _PH_W0, _PH_W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on uint32 arrays (broadcast); returns four uint32 arrays."""
    m32 = np.uint64(0xFFFFFFFF)
    c = [np.asarray(x, np.uint64) for x in (c0, c1, c2, c3)]
    k0, k1 = np.uint64(k0), np.uint64(k1)
    for _ in range(10):
        p0 = np.uint64(_PH_M0) * c[0]
        p1 = np.uint64(_PH_M1) * c[2]
        c = [((p1 >> np.uint64(32)) ^ c[1] ^ k0) & m32, p1 & m32, ((p0 >> np.uint64(32)) ^ c[3] ^ k1) & m32, p0 & m32]
        k0 = (k0 + np.uint64(_PH_W0)) & m32
        k1 = (k1 + np.uint64(_PH_W1)) & m32
    return [x.astype(np.uint32) for x in c]


def philox_uniforms(n: int, seed: int = 0, start: int = 0) -> np.ndarray:
    """(n, 18) uniforms in [0, 1) of pairs [start, start + n) (53-bit, numpy's recipe)."""
    ids = np.arange(start, start + n, dtype=np.uint64)
    lo, hi = (ids & np.uint64(0xFFFFFFFF)), ids >> np.uint64(32)
    k0, k1 = seed & 0xFFFFFFFF, ((seed >> 32) ^ 0x5EED) & 0xFFFFFFFF
    u = np.empty((n, 18))
    for call in range(9):
        r = philox4x32_10(lo, hi, np.full(n, call, np.uint64), np.zeros(n, np.uint64), k0, k1)
        for j in range(2):
            a, b = r[2 * j].astype(np.float64), r[2 * j + 1]
            u[:, 2 * call + j] = (np.floor(a / 32) * 67108864.0 + (b >> np.uint32(6))) / 9007199254740992.0
    return u


def philox_pairs(n: int, seed: int = 0, sep=(-0.05, 0.2), start: int = 0):
    """(A, B) (n, 3, 3) of the device generator (up to the last ulps of
    log / sincos / rsqrt, which CUDA and numpy round differently)."""
    u = philox_uniforms(n, seed, start)
    A = u[:, :9].reshape(n, 3, 3)
    r = np.sqrt(-2.0 * np.log(1.0 - u[:, 10::2]))
    th = 2.0 * np.pi * u[:, 11::2]
    z = np.empty((n, 8))
    z[:, 0::2] = r * np.cos(th)
    z[:, 1::2] = r * np.sin(th)
    q = z[:, :4] / np.linalg.norm(z[:, :4], axis=1, keepdims=True)
    v = z[:, 4:7] / np.linalg.norm(z[:, 4:7], axis=1, keepdims=True)
    s = sep[0] + (sep[1] - sep[0]) * u[:, 9]
    c = A.mean(axis=1, keepdims=True)
    return A, rotate_about(A, c, rotation_matrices(q), s[:, None] * v)
