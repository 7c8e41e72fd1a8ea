"""Shared helpers of the multiscale tests: scenes from tests/golden/ms_float*.npz."""

from __future__ import annotations

import numpy as np

from conftest import GOLDEN

SIDES = ("i", "j")


def load(real: str) -> dict:
    return dict(np.load(GOLDEN / f"ms_{real}.npz"))


def scenes(g: dict) -> list[str]:
    return [str(s) for s in g["scenes"]]


def tree(g: dict, scene: str, side: str) -> dict:
    t = {k: g[f"{scene}_{side}_{k}"] for k in ("tris", "eps", "child_off", "child_ids", "height")}
    t["n_nodes"] = int(g[f"{scene}_{side}_n_nodes"])
    return t


def moved(t: dict, R: np.ndarray, shift: np.ndarray) -> dict:
    """The same tree under an extra rigid motion (new coordinates, same topology)."""
    u = dict(t)
    x = t["tris"].reshape(-1, 3).astype(np.float64)
    u["tris"] = (x @ R.T + shift).astype(t["tris"].dtype).reshape(t["tris"].shape)
    return u
