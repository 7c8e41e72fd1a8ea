"""Golden fixtures for the multiscale traversal.

Runs in THIS container only: imports the read-only reference from
/root/reference/pkg/src, builds its own two-particle scenes (the shapes of
the reference's tests/test_stepping.py two_sphere_system and
test_asymmetric_unfolding), runs tricontact.stepping.multiscale_contacts
(RK/stepping.py:311-368) and single_level_contacts (:285-308) on them, and
writes per-scene FlatTree arrays (world coordinates under the particle's
motion, halos, children CSR, heights) with the reference's contacts, per-height
check counts and kernel counters.

    python tests/golden/make_multiscale_golden.py   # writes tests/golden/ms_float{64,32}.npz

The float32 fixture is produced in a child interpreter with
TRICONTACT_REAL=float32 (the reference fixes its scalar type at import).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")


def _flat_arrays(particle, motion):
    f = particle.flat
    child_off = np.zeros(f.tri.shape[0] + 1, np.int32)
    child_off[1:] = np.cumsum([c.size for c in f.children])
    child_ids = np.concatenate([c for c in f.children if c.size]).astype(np.int32)
    return dict(tris=particle.world_tris(motion).reshape(-1, 9), eps=f.eps.copy(), child_off=child_off,
                child_ids=child_ids, height=f.height.astype(np.int32), n_nodes=np.int64(f.n_nodes),
                local=f.tri.reshape(-1, 9).copy(),
                motion=np.concatenate([np.asarray(motion.rotation, np.float64),
                                       np.asarray(motion.translation, np.float64)]))


def _scene_out(prefix, system, out):
    from tricontact.kernels import KernelParams
    from tricontact.stepping import StepStats, multiscale_contacts, single_level_contacts

    pi, pj = system.particles[0], system.particles[1]
    params = KernelParams()
    stats = StepStats()
    multi = multiscale_contacts(pi, pj, (0, 1), params, stats)
    single = single_level_contacts(pi, pj, (0, 1), params, StepStats())
    for side, p in (("i", pi), ("j", pj)):
        for k, v in _flat_arrays(p, p.motion).items():
            out[f"{prefix}_{side}_{k}"] = v
    out[f"{prefix}_source"] = np.array([c.source for c in multi], np.int64).reshape(-1, 2)
    out[f"{prefix}_position"] = np.array([c.position for c in multi]).reshape(-1, 3)
    out[f"{prefix}_normal"] = np.array([c.normal for c in multi]).reshape(-1, 3)
    out[f"{prefix}_eps"] = np.array([c.eps for c in multi], np.float64).reshape(-1, 2)
    hmax = max(stats.checks_by_level) if stats.checks_by_level else 0
    out[f"{prefix}_checks"] = np.array([stats.checks_by_level.get(h, 0) for h in range(hmax + 1)], np.int64)
    k = stats.kernel
    out[f"{prefix}_counters"] = np.array([k.iterative_invocations, k.comparison_invocations,
                                          k.fallback_invocations], np.int64)
    out[f"{prefix}_single_source"] = np.array([c.source for c in single], np.int64).reshape(-1, 2)
    out[f"{prefix}_single_position"] = np.array([c.position for c in single]).reshape(-1, 3)
    out[f"{prefix}_single_normal"] = np.array([c.normal for c in single]).reshape(-1, 3)
    out[f"{prefix}_single_eps"] = np.array([pi.epsilon, pj.epsilon], np.float64)
    print(prefix, "contacts", len(multi), "single", len(single), "checks", out[f"{prefix}_checks"].tolist(),
          flush=True)


def _find_contacts_cases(out):
    """RK/contact.py:97-140 find_contacts_single_level: two soups with unequal
    halos, a soup against itself (diagonal skipped), ragged sizes."""
    from tricontact.contact import find_contacts_single_level
    from tricontact.geometry import flatten
    from tricontact.kernels import KernelCounters, KernelParams
    from tricontact.scenes import SceneSpec, build_scene
    from tricontact.stepping import system_from_scene

    spec = SceneSpec(kind="ParticleParticle", triangle_count=80, initial_gap=1e-3, approach_speed=0.5,
                     seed=3, relative_tilt_deg=10.0)
    sysm = system_from_scene(build_scene(spec), KernelParams())
    wi = sysm.particles[0].world_tris().reshape(-1, 3, 3)[sysm.particles[0].flat.n_nodes:]
    wj = sysm.particles[1].world_tris().reshape(-1, 3, 3)[sysm.particles[1].flat.n_nodes:]
    plane = system_from_scene(build_scene(SceneSpec(kind="ParticleOnPlane", triangle_count=80, drop_height=0.0)),
                              KernelParams())
    pl = [p.world_tris().reshape(-1, 3, 3)[p.flat.n_nodes:] for p in plane.particles]
    soup = flatten(wi)
    cases = {
        "two": (flatten(wi), flatten(wj), 1e-2, 2e-2),
        "self": (soup, soup, None, None),
        "ragged": (flatten(pl[0]), flatten(pl[1]), None, None),
        "ragged_t": (flatten(pl[1]), flatten(pl[0]), 5e-3, 1e-2),
    }
    names = []
    for name, (si, sj, ei, ej) in cases.items():
        counters = KernelCounters()
        res = find_contacts_single_level(si, sj, KernelParams(), counters, pair=(3, 7), eps_i=ei, eps_j=ej)
        pre = f"fc_{name}"
        names.append(name)
        out[f"{pre}_tris_i"] = si.triangles().reshape(-1, 9).copy()
        out[f"{pre}_tris_j"] = sj.triangles().reshape(-1, 9).copy()
        out[f"{pre}_same"] = np.bool_(si is sj)
        out[f"{pre}_eps"] = np.array([np.nan if ei is None else ei, np.nan if ej is None else ej])
        out[f"{pre}_source"] = np.array([c.source for c in res], np.int64).reshape(-1, 2)
        out[f"{pre}_position"] = np.array([c.position for c in res]).reshape(-1, 3)
        out[f"{pre}_normal"] = np.array([c.normal for c in res]).reshape(-1, 3)
        out[f"{pre}_counters"] = np.array([counters.iterative_invocations, counters.comparison_invocations,
                                           counters.fallback_invocations], np.int64)
        print(pre, "contacts", len(res), flush=True)
    out["fc_cases"] = np.array(names)


def _tree_arrays(tree, pre, out):
    nodes = list(tree.nodes())
    index = {id(n): k for k, n in enumerate(nodes)}
    out[f"{pre}_node_tri"] = np.stack([np.asarray(n.triangle, np.float64).reshape(3, 3) for n in nodes])
    out[f"{pre}_node_eps"] = np.array([float(n.epsilon) for n in nodes])
    out[f"{pre}_node_leaf"] = np.array([n.is_leaf for n in nodes])
    kids = [np.array([index[id(c)] for c in n.children], np.int64) for n in nodes]
    leaves = [np.asarray(n.leaf_indices(), np.int64) for n in nodes]
    for name, lists in (("kids", kids), ("leafidx", leaves)):
        off = np.zeros(len(nodes) + 1, np.int64)
        off[1:] = np.cumsum([a.size for a in lists])
        out[f"{pre}_{name}_off"] = off
        out[f"{pre}_{name}"] = np.concatenate(lists) if off[-1] else np.zeros(0, np.int64)
    out[f"{pre}_finest"] = np.float64(tree.finest_epsilon)


def _surrogate_cases(out):
    """RK/surrogate.py:237-257 conservative_epsilon and :463-505
    validate_conservative on reference-built trees."""
    from tricontact.geometry import triangle
    from tricontact.kernels import KernelParams
    from tricontact.scenes import SceneSpec, build_scene
    from tricontact.stepping import system_from_scene
    from tricontact.surrogate import build_surrogate_tree, conservative_epsilon, validate_conservative

    rng = np.random.default_rng(99)
    for count in (80, 320):
        spec = SceneSpec(kind="ParticleParticle", triangle_count=count, initial_gap=1e-3, approach_speed=0.5,
                         seed=3, relative_tilt_deg=10.0)
        p = system_from_scene(build_scene(spec), KernelParams()).particles[0]
        mesh = p.body_tris.reshape(-1, 3, 3)
        tree = build_surrogate_tree(mesh, 8, seed=0)
        pre = f"sg{count}"
        out[f"{pre}_mesh"] = mesh.reshape(-1, 9).copy()
        _tree_arrays(tree, pre, out)
        for spt in (10, 3):
            r = validate_conservative(tree, mesh, samples_per_triangle=spt)
            out[f"{pre}_valid_{spt}"] = np.array([r["worst_slack"], float(r["ok"]), r["checked_nodes"]])
        tree.root.epsilon *= 0.5
        r = validate_conservative(tree, mesh)
        out[f"{pre}_halved_valid"] = np.array([r["worst_slack"], float(r["ok"]), r["checked_nodes"]])
        print(pre, "nodes", out[f"{pre}_valid_10"], out[f"{pre}_halved_valid"], flush=True)
    ce = []
    t = triangle([0, 0, 0], [1, 0, 0], [0, 1, 0])
    cases = [(t, t[None], 0.25), (t, (t + np.array([0, 0, 0.7]))[None], 0.0)]
    for _ in range(6):
        cases.append((rng.normal(size=(3, 3)), rng.normal(scale=0.6, size=(12, 3, 3)), rng.uniform(0.01, 0.1, 12)))
    for k, (sur, ch, e) in enumerate(cases):
        out[f"ce{k}_surrogate"] = np.asarray(sur, np.float64)
        out[f"ce{k}_children"] = np.asarray(ch, np.float64).reshape(-1, 9)
        out[f"ce{k}_eps"] = np.asarray(e, np.float64)
        ce.append(conservative_epsilon(sur, ch, e))
    out["ce_values"] = np.array(ce)


def run() -> dict:
    from tricontact.geometry import RigidMotion
    from tricontact.kernels import KernelParams
    from tricontact.scenes import SceneSpec, build_scene
    from tricontact.stepping import system_from_scene

    out = {}
    rng = np.random.default_rng(20261020)
    for count, poses in ((80, 4), (320, 3)):
        spec = SceneSpec(kind="ParticleParticle", triangle_count=count, initial_gap=1e-3, approach_speed=0.5,
                         seed=3, relative_tilt_deg=10.0)
        system = system_from_scene(build_scene(spec), KernelParams())
        _scene_out(f"s{count}_rest", system, out)
        rest = system.particles[1].motion.translation.copy()
        for k in range(poses):
            # random orientation of particle j at a slightly perturbed rest offset
            system.particles[1].motion = RigidMotion.random_rotation(
                rng, translation=rest * (1.0 + rng.uniform(-2e-2, 5e-3)))
            _scene_out(f"s{count}_p{k}", system, out)
    spec = SceneSpec(kind="ParticleOnPlane", triangle_count=80, drop_height=0.0)
    _scene_out("plane", system_from_scene(build_scene(spec), KernelParams()), out)
    _find_contacts_cases(out)
    _surrogate_cases(out)
    out["scenes"] = np.array(sorted({k.split("_")[0] + "_" + k.split("_")[1] if not k.startswith("plane") else "plane"
                                     for k in out if k.endswith("_checks")}))
    return out


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--worker":
        sys.path.insert(0, str(REF_SRC))
        np.savez_compressed(sys.argv[2], **run())
        return
    for real in ("float64", "float32"):
        env = dict(os.environ, TRICONTACT_REAL=real, PYTHONPATH=str(REF_SRC))
        dst = HERE / f"ms_{real}.npz"
        subprocess.run([sys.executable, __file__, "--worker", str(dst)], env=env, check=True)
        print("wrote", dst, dst.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
