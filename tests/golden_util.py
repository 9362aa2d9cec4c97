"""Load tests/golden fixtures (made by tests/golden/make_golden.py from the
reference package) into this repo's host structures."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
SCHEMES = ["m1-double", "m1-single", "m1-mixed", "m2-double", "m2-single", "m2-mixed",
           "m3:c=-1", "m3:c=1", "m3:c=3", "m3:c=5", "m3:c=7"]
FP64_ONLY = {"m1-double", "m2-double", "m3:c=7"}   # all-FP64 payloads at these fixtures


def load(name: str):
    arr = dict(np.load(GOLDEN / f"{name}.npz"))
    meta = json.loads((GOLDEN / f"{name}.json").read_text())
    return arr, meta


def hmatrix_from_fixture(arr):
    """The reference's H-matrix (exact FP64 masters) as this repo's HMatrixF64."""
    from paper_1911_00093_b200.compress import HMatrixF64, PackedMaster
    from paper_1911_00093_b200.partition import BlockPartition, ClusterNode, ClusterTree

    table = arr["table"]
    n = int(arr["perm"].shape[0])
    sizes = np.where(arr["kinds"] == 0, (table[:, 1] - table[:, 0]) * (table[:, 3] - table[:, 2]),
                     arr["ranks"] * ((table[:, 1] - table[:, 0]) + (table[:, 3] - table[:, 2])))
    offsets = np.zeros(table.shape[0], dtype=np.int64)
    offsets[1:] = np.cumsum(sizes)[:-1]
    root = ClusterNode(0, n, np.zeros(3), np.zeros(3))
    tree = ClusterTree(root=root, permutation=arr["perm"], leaf_size=n)
    part = BlockPartition(n=n, tree=tree, table=table)
    pm = PackedMaster(np.ascontiguousarray(arr["data"]), arr["kinds"].astype(np.int32),
                      arr["ranks"].astype(np.int64), offsets)
    return HMatrixF64(part, packed=pm)


def config1_hmatrix():
    """Config 1 rebuilt with this repo's builder (same mesh recipe)."""
    import paper_1911_00093_b200 as hx
    mesh = hx.jittered_sphere_mesh(3, seed=42)
    return mesh, hx.build_hmatrix(mesh, aca_tol=1e-4, leaf_size=32, eta=2.0)


def fingerprint(h) -> dict:
    """Cheap identity of an H-matrix: sha256 of the block table and ranks, and
    order-sensitive 64-bit checksums of every stored FP64 master value (used
    to assert that a test solves the matrix a golden file was made on)."""
    import hashlib
    pm = h.packed
    tab = np.ascontiguousarray(h.partition.table, dtype=np.int64)
    d = hashlib.sha256(tab.tobytes())
    d.update(np.ascontiguousarray(pm.ranks, dtype=np.int64).tobytes())
    bits = np.ascontiguousarray(pm.data).view(np.uint64)
    w = (np.arange(bits.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    with np.errstate(over="ignore"):
        mix = int(np.bitwise_xor.reduce(bits * w)) if bits.size else 0
        tot = int(np.add.reduce(bits, dtype=np.uint64)) if bits.size else 0
    return {"table_ranks_sha256": d.hexdigest(), "data_xor_mix": f"{mix:016x}",
            "data_sum": f"{tot:016x}", "n_values": int(bits.size)}
