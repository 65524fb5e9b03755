"""GPU: every probe path of k_aot (warp bitmap, warp rank bitmap, warp hash --
two-choice buckets, and the linear-probing fallback --, CTA bitmap, CTA rank
bitmap, CTA hash, global binary search) against the oracle.  The full configs reach the wide-window paths only at scale, so this
test runs tools/sanitize_run.py's parity workload (every kernel x mode x
order, partitions, device verification) on a build of the library whose
probe regions are shrunk (paper_2006_11494_b200/_build.py VARIANTS["paths"]),
where small graphs exercise all of them (variants: rank bitmap on / off,
bucket hashes forced to fail over to linear probing), and checks from the
path diagnostics (TL_DEBUG_PATHS) that each path carried work."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATHS = ("warp-bitmap", "warp-rank", "warp-hash", "cta-bitmap", "cta-rank", "cta-hash", "global")


def test_every_probe_path_matches_oracle(built):
    from paper_2006_11494_b200 import _build

    work = dict.fromkeys(PATHS, 0)
    for variant in ("paths", "paths_hash", "paths_fallback"):
        lib = _build.build_variant(variant)
        env = dict(os.environ, TL_LIB_PATH=lib, TL_DEBUG_PATHS="1")
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--size", "medium"],
                           env=env, capture_output=True, text=True, timeout=1200)
        assert p.returncode == 0, (variant, p.stderr[-3000:])
        assert "ingest ok" in p.stdout
        for line in p.stderr.splitlines():
            if line.startswith("[tl paths]"):
                for name in PATHS:
                    work[name] += int(re.search(rf"{name} (\d+)", line).group(1))
    assert all(work[k] > 0 for k in PATHS), work


@pytest.mark.parametrize("variant", ["ring_tma", "ring_ldgsts"])
def test_async_staging_variants_match_oracle(built, variant):
    """The measured-and-rejected staging of long windows through a per-warp
    shared-memory ring (TL_RING=1 bulk copies via the TMA engine,
    TL_RING=2 per-thread cp.async) stays parity-green on the same workload."""
    from paper_2006_11494_b200 import _build

    lib = _build.build_variant(variant)
    env = dict(os.environ, TL_LIB_PATH=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--size", "medium"],
                       env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, (variant, p.stderr[-3000:])
    assert "rmat17 ok" in p.stdout and "ingest ok" in p.stdout

