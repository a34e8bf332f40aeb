"""Structural checks of a flat BVH (test helper; the invariants the
reference's builder guarantees, hrpp/bvh.py:184-357 / :448-476)."""

import numpy as np


def check_bvh(b, bounds_eps: float = 1e-5) -> None:
    """Assert that ``b`` is a DFS-preorder binary tree rooted at 0 whose
    children nest in their parents' boxes, whose leaves tile the triangle
    slots exactly once and whose max_depth is the deepest leaf's depth."""
    n = b.node_count
    inner = np.flatnonzero(b.left >= 0)
    leaves = np.flatnonzero(b.left < 0)
    # every non-root node has exactly one parent, which lists it as a child
    kids = np.concatenate([b.left[inner], b.right[inner]])
    assert kids.min(initial=1) >= 1 and kids.max(initial=0) < n
    assert np.array_equal(np.sort(kids), np.arange(1, n)), "not a tree over all nodes"
    assert np.array_equal(b.left[inner], inner + 1), "left child is not parent + 1"
    for c in (b.left[inner], b.right[inner]):
        assert np.array_equal(b.parent[c], inner)
        assert np.array_equal(b.depth[c], b.depth[inner] + 1)
        assert np.all(b.bmin[c] >= b.bmin[inner] - bounds_eps)
        assert np.all(b.bmax[c] <= b.bmax[inner] + bounds_eps)
    assert int(b.parent[0]) < 0 and int(b.depth[0]) == 0
    # leaves: non-empty, disjoint, covering [0, triangle_count)
    assert np.all(b.count[leaves] >= 1)
    cover = np.zeros(b.triangle_count + 1, np.int64)
    np.add.at(cover, b.first[leaves], 1)
    np.add.at(cover, b.first[leaves] + b.count[leaves], -1)
    assert np.all(np.cumsum(cover)[:-1] == 1), "leaf slot ranges must tile the slots once"
    assert b.max_depth == int(b.depth[leaves].max())
