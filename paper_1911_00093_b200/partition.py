"""Cluster tree and admissible block partition (host, untimed).

Interface of reference pkg/src/hmx/partition.py:16-25; the tree and the
dual traversal run in the native builder (csrc/hbuild.cpp) because the
reference's Python recursion dominates set-up time at N >= 81,920.  The
emitted block list is identical, in the same order, to the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native

__all__ = [
    "ClusterNode",
    "ClusterTree",
    "Block",
    "BlockPartition",
    "build_cluster_tree",
    "build_block_partition",
    "is_admissible",
    "dump_partition",
]

DEFAULT_LEAF_SIZE = 32   # reference partition.py:27
DEFAULT_ETA = 2.0        # reference partition.py:28


@dataclass
class ClusterNode:
    """Index range [start, end) of permuted indices plus its bounding box."""

    start: int
    end: int
    bbox_min: np.ndarray
    bbox_max: np.ndarray
    left: "ClusterNode | None" = None
    right: "ClusterNode | None" = None

    @property
    def is_leaf(self) -> bool:
        return self.left is None

    @property
    def size(self) -> int:
        return self.end - self.start

    @property
    def diameter(self) -> float:
        return float(np.linalg.norm(self.bbox_max - self.bbox_min))


def node_distance(a: ClusterNode, b: ClusterNode) -> float:
    """Euclidean distance between two cluster bounding boxes (reference partition.py:56-60)."""
    gap = np.maximum(0.0, np.maximum(a.bbox_min - b.bbox_max, b.bbox_min - a.bbox_max))
    return float(np.linalg.norm(gap))


@dataclass
class ClusterTree:
    """Cluster tree over the panels and its permutation (reference partition.py:63-72)."""
    root: ClusterNode
    permutation: np.ndarray  # permuted index -> original panel index
    leaf_size: int
    nodes: np.ndarray | None = field(default=None, repr=False)  # native node table

    @property
    def n(self) -> int:
        return self.root.end


@dataclass(frozen=True)
class Block:
    """Half-open row/col ranges in permuted indices, plus admissibility."""

    row_start: int
    row_end: int
    col_start: int
    col_end: int
    admissible: bool

    @property
    def rows(self) -> int:
        return self.row_end - self.row_start

    @property
    def cols(self) -> int:
        return self.col_end - self.col_start


class BlockPartition:
    """Ordered block list.  Backed by an (nb, 5) int64 table; the list of
    `Block` objects is materialised on first access."""

    def __init__(self, blocks=None, n: int = 0, tree: ClusterTree | None = None, table=None):
        self.n = int(n)
        self.tree = tree
        if table is None:
            blocks = list(blocks or [])
            table = np.array([[b.row_start, b.row_end, b.col_start, b.col_end,
                               1 if b.admissible else 0] for b in blocks],
                             dtype=np.int64).reshape(-1, 5)
            self._blocks = blocks
        else:
            self._blocks = None
        self.table = np.ascontiguousarray(table, dtype=np.int64)

    @property
    def blocks(self) -> list:
        if self._blocks is None:
            self._blocks = [Block(int(r[0]), int(r[1]), int(r[2]), int(r[3]), bool(r[4]))
                            for r in self.table.tolist()]
        return self._blocks

    def __len__(self):
        return int(self.table.shape[0])

    @property
    def admissible_blocks(self) -> list:
        return [b for b in self.blocks if b.admissible]

    def coverage_count(self) -> int:
        t = self.table
        return int(np.sum((t[:, 1] - t[:, 0]) * (t[:, 3] - t[:, 2])))


def _node_array(tree_nodes: np.ndarray):
    return tree_nodes.ctypes.data_as(ctypes.c_void_p)


_NODE_DTYPE = np.dtype([("start", np.int64), ("end", np.int64), ("bmin", np.float64, 3),
                        ("bmax", np.float64, 3), ("left", np.int64), ("right", np.int64)])
assert _NODE_DTYPE.itemsize == ctypes.sizeof(_native.HbNode)


def build_cluster_tree(mesh, leaf_size: int = DEFAULT_LEAF_SIZE) -> ClusterTree:
    """Median-bisection tree over `mesh.centroids` (reference partition.py:74-105)."""
    pts = np.ascontiguousarray(mesh.centroids, dtype=np.float64)
    n = pts.shape[0]
    if n < 1:
        raise ValueError("cannot build a tree over an empty mesh")
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    perm = np.empty(n, dtype=np.int64)
    cap = 2 * n
    nodes = np.zeros(cap, dtype=_NODE_DTYPE)
    count = ctypes.c_int64(0)
    rc = _native.host().hb_cluster_tree(_native.ptr(pts, _native.c_f64p), n, int(leaf_size),
                                         _native.ptr(perm, _native.c_i64p), _node_array(nodes),
                                         cap, ctypes.byref(count))
    if rc != 0:
        raise RuntimeError(f"cluster tree construction failed ({rc})")
    nodes = nodes[: count.value].copy()
    objs = [ClusterNode(int(r["start"]), int(r["end"]), r["bmin"].copy(), r["bmax"].copy())
            for r in nodes]
    for k, r in enumerate(nodes):
        if r["left"] >= 0:
            objs[k].left = objs[int(r["left"])]
            objs[k].right = objs[int(r["right"])]
    perm.setflags(write=False)
    return ClusterTree(root=objs[0], permutation=perm, leaf_size=int(leaf_size), nodes=nodes)


def _tree_table(tree: ClusterTree) -> np.ndarray:
    if tree.nodes is not None:
        return tree.nodes
    order, index = [], {}

    def walk(node):
        index[id(node)] = len(order)
        order.append(node)
        if not node.is_leaf:
            walk(node.left)
            walk(node.right)

    walk(tree.root)
    nodes = np.zeros(len(order), dtype=_NODE_DTYPE)
    for k, nd in enumerate(order):
        nodes[k]["start"], nodes[k]["end"] = nd.start, nd.end
        nodes[k]["bmin"], nodes[k]["bmax"] = nd.bbox_min, nd.bbox_max
        nodes[k]["left"] = -1 if nd.is_leaf else index[id(nd.left)]
        nodes[k]["right"] = -1 if nd.is_leaf else index[id(nd.right)]
    return nodes


def is_admissible(s: ClusterNode, t: ClusterNode, eta: float) -> bool:
    """min(diam) <= eta * dist with dist > 0 (reference partition.py:142-148)."""
    dist = node_distance(s, t)
    return dist > 0.0 and min(s.diameter, t.diameter) <= eta * dist


def build_block_partition(tree: ClusterTree, eta: float = DEFAULT_ETA) -> BlockPartition:
    """Dual traversal from (root, root) (reference partition.py:151-169)."""
    if eta <= 0.0:
        raise ValueError("eta must be positive")
    nodes = _tree_table(tree)
    lib = _native.host()
    count = int(lib.hb_partition(_node_array(nodes), nodes.shape[0], float(eta), None, 0))
    table = np.empty((count, 5), dtype=np.int64)
    got = int(lib.hb_partition(_node_array(nodes), nodes.shape[0], float(eta),
                               _native.ptr(table, _native.c_i64p), count))
    if got != count:
        raise RuntimeError("partition traversal is not deterministic")
    return BlockPartition(n=tree.n, tree=tree, table=table)


def dump_partition(partition: BlockPartition, path) -> None:
    """`i_s i_e j_s j_e admissible` per block (reference partition.py:172-177)."""
    with open(path, "w", encoding="ascii") as fh:
        for r in partition.table.tolist():
            fh.write(f"{r[0]} {r[1]} {r[2]} {r[3]} {r[4]}\n")
