"""C2 (R-MAT s20, 4.24e8 triangles) compared DIRECTLY against the
reference's own listing, run in the same test on the GPU box's host
(SURVEY.md §8d, Appendix B item 2):

  reference: Graph::from_edges -> degree_order -> orient ->
             run_parallel_collecting(aot, {threads, 64}) (parallel.cpp:10-17),
             canonicalised and sorted on the host (canonicalize_emissions,
             engine.cpp:51-57, as numpy);
  B200:      tl_run_list(canonical=1): device listing + canonicalisation +
             lexicographic sort, downloaded.

The two sorted canonical lists (5.1 GB each as triples) must be identical
element for element; the raw role-order emissions must be the same multiset.
"""
import numpy as np
import pytest

import oracle as O
from paper_2006_11494_b200 import capi
from paper_2006_11494_b200.configs import CONFIGS

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _pack(tri: np.ndarray) -> np.ndarray:
    """Canonical triples (a < b < c < 2^21) as one sortable uint64 key."""
    t = tri.astype(np.uint64)
    return (t[:, 0] << np.uint64(42)) | (t[:, 1] << np.uint64(21)) | t[:, 2]


def test_c2_sorted_set_equals_reference_collecting(golden):
    import torch

    cfg = CONFIGS["c2"]
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    pairs = d.cpu().numpy().view(np.uint32).reshape(-1, 2)
    do = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"]).orient()
    del d
    torch.cuda.empty_cache()
    assert cfg["n"] <= 1 << 21

    st, ours = do.list(canonical=True)  # device canonicalise + sort
    assert st["triangles"] == golden["c2"]["triangles"]
    ours_keys = _pack(ours)
    del ours

    ref = O.RefGraph(cfg["n"], pairs)
    del pairs
    rst, raw = ref.collect(threads=O.hardware_threads())
    assert rst["triangles"] == st["triangles"] == raw.shape[0]
    canon = np.sort(raw, axis=1)  # canonical_triangle (graph.cpp:148-153)
    ref_keys = _pack(canon)
    del canon
    ref_keys.sort(kind="stable")
    assert np.array_equal(ref_keys, ours_keys)  # identical sorted canonical lists, element for element
    assert np.all(ref_keys[1:] > ref_keys[:-1])  # no duplicate emission on either side
    del ref_keys, ours_keys

    # raw role order (pivot, neighbor, witness): the same emissions as a multiset
    _, ours_raw = do.list(canonical=False)
    a = (ours_raw[:, 0].astype(np.uint64) << np.uint64(42)) | (ours_raw[:, 1].astype(np.uint64) << np.uint64(21)) | \
        ours_raw[:, 2].astype(np.uint64)
    b = (raw[:, 0].astype(np.uint64) << np.uint64(42)) | (raw[:, 1].astype(np.uint64) << np.uint64(21)) | \
        raw[:, 2].astype(np.uint64)
    a.sort()
    b.sort()
    assert np.array_equal(a, b)
    for k in ("probes", "table_builds", "positive_triangles", "negative_triangles"):
        assert st[k] == rst[k], k
