"""Host-side mesh plumbing (numpy): the data the hot path consumes.

This mirrors the reference's `Mesh` (/root/reference/proj/include/hbflow/mesh.hpp:16-60)
and `Mesh::finalize` (src/mesh.cpp:60-157): element orientation, boundary
facets with outward normals and areas, and the Dirichlet node mask.  It is
out-of-scope plumbing ("reused host plumbing; its outputs are
hot-path inputs"); element geometry (mesh.cpp:159-203) is computed on the GPU
by the library (hbgpu_create) because every element kernel reads it.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DIRICHLET = 0
NEUMANN = 1


class GeometryError(RuntimeError):
    """Degenerate or inconsistent geometry (errors.hpp:17-22)."""


class ParseError(RuntimeError):
    """Malformed input (errors.hpp:9-14)."""


@dataclass
class Patch:
    name: str
    kind: int  # DIRICHLET | NEUMANN
    facets: np.ndarray  # (F,3) int32, oriented after finalize
    normals: np.ndarray | None = None  # (F,3) unit outward
    areas: np.ndarray | None = None  # (F,)

    @property
    def area(self) -> float:
        return float(self.areas.sum()) if self.areas is not None else 0.0


@dataclass
class Mesh:
    xyz: np.ndarray  # (nn,3) float64
    conn: np.ndarray  # (ne,4) int32
    patches: list[Patch] = field(default_factory=list)
    dirichlet: np.ndarray | None = None  # (nn,) uint8

    @property
    def num_nodes(self) -> int:
        return int(self.xyz.shape[0])

    @property
    def num_elements(self) -> int:
        return int(self.conn.shape[0])

    def patch_index(self, name: str) -> int:
        for k, p in enumerate(self.patches):
            if p.name == name:
                return k
        return -1

    def finalize(self) -> "Mesh":
        """Orientation, boundary normals/areas, Dirichlet mask (mesh.cpp:60-157)."""
        xyz = np.ascontiguousarray(self.xyz, dtype=np.float64)
        conn = np.ascontiguousarray(self.conn, dtype=np.int32).copy()
        nn = xyz.shape[0]
        if conn.size and (conn.min() < 0 or conn.max() >= nn):
            raise ParseError("element references a node out of range")
        x0, x1, x2, x3 = (xyz[conn[:, k]] for k in range(4))
        vol = np.einsum("ij,ij->i", x1 - x0, np.cross(x2 - x0, x3 - x0)) / 6.0
        neg = vol < 0.0
        conn[neg, 1], conn[neg, 2] = conn[neg, 2].copy(), conn[neg, 1].copy()
        if not np.all(np.abs(vol) > 0.0):
            raise GeometryError("degenerate element with zero volume")

        # Boundary faces = element faces seen once (mesh.cpp:92-111).
        faces = np.concatenate(
            [conn[:, [1, 2, 3]], conn[:, [0, 3, 2]], conn[:, [0, 1, 3]], conn[:, [0, 2, 1]]]
        )
        opp = np.concatenate([conn[:, 0], conn[:, 1], conn[:, 2], conn[:, 3]])
        keys = np.sort(faces, axis=1).astype(np.int64)
        code = (keys[:, 0] * nn + keys[:, 1]) * nn + keys[:, 2]
        uniq, first, counts = np.unique(code, return_index=True, return_counts=True)
        bmask = counts == 1
        bcode = uniq[bmask]
        bopp = opp[first[bmask]]

        claimed = 0
        for p in self.patches:
            f = np.ascontiguousarray(p.facets, dtype=np.int32).copy()
            if f.size and (f.min() < 0 or f.max() >= nn):
                raise ParseError(f"patch '{p.name}' references node out of range")
            fk = np.sort(f, axis=1).astype(np.int64)
            fcode = (fk[:, 0] * nn + fk[:, 1]) * nn + fk[:, 2]
            pos = np.searchsorted(bcode, fcode)
            pos = np.minimum(pos, max(len(bcode) - 1, 0))
            if len(bcode) == 0 or not np.all(bcode[pos] == fcode):
                raise GeometryError(f"patch '{p.name}' facet is not a boundary face")
            a, b, c = xyz[f[:, 0]], xyz[f[:, 1]], xyz[f[:, 2]]
            nv = np.cross(b - a, c - a)
            ln = np.sqrt(np.einsum("ij,ij->i", nv, nv))
            if not np.all(ln > 0.0):
                raise GeometryError(f"zero-area facet in patch '{p.name}'")
            nv = nv / ln[:, None]
            o = xyz[bopp[pos]]
            flip = np.einsum("ij,ij->i", nv, o - a) > 0.0
            nv[flip] = -nv[flip]
            f[flip, 1], f[flip, 2] = f[flip, 2].copy(), f[flip, 1].copy()
            p.facets, p.normals, p.areas = f, nv, 0.5 * ln
            claimed += len(f)
        if self.patches and claimed != len(bcode):
            raise GeometryError(
                f"patches do not cover the boundary: {len(bcode) - claimed} unclaimed facets"
            )
        dmask = np.zeros(nn, dtype=np.uint8)
        for p in self.patches:
            if p.kind == DIRICHLET:
                dmask[p.facets.reshape(-1)] = 1
        self.xyz, self.conn, self.dirichlet = xyz, conn, dmask
        return self

    def characteristic_length(self) -> float:
        """h_c = (6 sqrt(2) Vbar)^(1/3) (mesh.cpp:213-224)."""
        x0, x1, x2, x3 = (self.xyz[self.conn[:, k]] for k in range(4))
        vol = np.einsum("ij,ij->i", x1 - x0, np.cross(x2 - x0, x3 - x0)) / 6.0
        return float(np.cbrt(6.0 * np.sqrt(2.0) * vol.mean()))


def boundary_faces(conn: np.ndarray, nn: int) -> np.ndarray:
    """Element faces seen exactly once, unoriented (F,3)."""
    faces = np.concatenate(
        [conn[:, [1, 2, 3]], conn[:, [0, 3, 2]], conn[:, [0, 1, 3]], conn[:, [0, 2, 1]]]
    )
    keys = np.sort(faces, axis=1).astype(np.int64)
    code = (keys[:, 0] * nn + keys[:, 1]) * nn + keys[:, 2]
    _, first, counts = np.unique(code, return_index=True, return_counts=True)
    return faces[first[counts == 1]].astype(np.int32)
