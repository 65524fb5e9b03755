"""CPU: the C-ABI library loads, exports every symbol include/trilist_b200.h
declares, validates arguments before touching a device, fails loudly (no CPU
fallback) without one, and its host-side pieces match the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2006_11494_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "trilist_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"TL_API\s+[\w\s\*]+?\b(tl_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(capi.EXPORTS)


def test_library_exports_every_declared_symbol(built):
    lib = C.CDLL(capi.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_only_the_c_abi_is_exported(built):
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert syms == set(declared_symbols())


def test_argument_validation_precedes_device_use(built):
    L = capi.lib()
    out = C.c_void_p()
    assert L.tl_graph_from_pairs(None, 5, 0, 0, 0, None, C.byref(out)) == capi.TL_EINVAL
    assert "pairs is NULL" in L.tl_last_error().decode()
    assert L.tl_graph_info(None, None, None, None, None) == capi.TL_EINVAL
    assert L.tl_aot_count(None, None, None) == capi.TL_EINVAL
    assert L.tl_chung_lu_prefix(1, 4, 32.0, 0.5, None) == capi.TL_EINVAL


def test_no_cpu_fallback_without_a_device(built):
    if capi.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(capi.TlError) as e:
        capi.DeviceGraph.from_pairs(np.array([[0, 1], [1, 2], [0, 2]], np.uint32), 3)
    assert e.value.code == capi.TL_ENODEV


def test_chung_lu_weights_match_oracle(built):
    import oracle as O

    for seed, n in ((3, 1000), (7, 4096)):
        assert np.array_equal(capi.chung_lu_prefix(seed, n, 32.0, 2.1), O.chung_lu_prefix(seed, n, 32.0, 2.1))


def test_version_string(built):
    assert "sm_100a" in capi.version()


def test_python_binding_mirrors_reference_names(built):
    from paper_2006_11494_b200 import trilist

    reference_names = {"ALGORITHMS", "Graph", "OrientedGraph", "ParseFailure", "brute_force_triangles", "cost_model",
                       "count_triangles", "edge_polarity", "list_triangles", "orient", "run", "verify_equivalence"}
    assert reference_names <= set(trilist.__all__)
    assert trilist.ALGORITHMS == ["cf", "cf-hash", "kclist", "aot"]
    assert trilist.REFERENCE_ALGORITHMS == ["cf", "cf-hash", "kclist", "aot"]
    assert issubclass(trilist.ParseFailure, ValueError)
    g = trilist.Graph()
    assert (g.num_vertices, g.num_edges) == (0, 0)


def test_async_staging_variants_carry_their_instructions():
    """SASS of the ring variants (built here, no GPU needed): the TMA ring's
    count kernel issues bulk copies (UBLKCP) completed on mbarriers
    (SYNCS.ARRIVE.TRANS64 / SYNCS.PHASECHK), the cp.async ring LDGSTS with
    zero fill; the product build has neither in its count kernel."""
    import subprocess

    from paper_2006_11494_b200 import _build

    def sass(lib):
        return subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                              text=True).stdout

    tma = sass(_build.build_variant("ring_tma"))
    assert "UBLKCP.S.G" in tma and "SYNCS.ARRIVE.TRANS64" in tma and "SYNCS.PHASECHK.TRANS64" in tma
    ldgsts = sass(_build.build_variant("ring_ldgsts"))
    assert "LDGSTS.E.BYPASS.128.ZFILL" in ldgsts
    prod = sass(_build.build_lib())
    assert "UBLKCP" not in prod and "LDGSTS" not in prod
