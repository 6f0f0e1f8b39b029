"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol
that include/gmaf.h declares; struct layouts of the binding match the header; the
workspace sizing and argument validation need no GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    from paper_2511_06824_b200 import build as B
    B.build()
    import paper_2511_06824_b200 as P
    return P


def _declared():
    hdr = open(os.path.join(ROOT, "include", "gmaf.h")).read()
    return sorted(set(re.findall(r"\b(gmaf_[a-z0-9_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(pkg):
    L = pkg.lib()
    names = _declared()
    assert "gmaf_solve" in names and "gmaf_create" in names
    for n in names:
        assert hasattr(L, n), n
    assert set(pkg.ABI_SYMBOLS) <= set(names)


def test_version_and_sizes(pkg):
    assert b"sm_100a" in pkg.lib().gmaf_version()
    import gmaf_inputs as gi
    g = pkg.make_grid(gi.grid(2048, 1024, "short"))
    nb = pkg.gmaf_workspace_bytes(g, 9)
    n = 2048 * 1024 * 9 * 8
    assert 9 * n <= nb <= 9 * n + (64 << 20)      # 9 fields of K*n doubles + small state
    assert C.sizeof(pkg.gmaf_condition) == 13 * 8
    assert C.sizeof(pkg.gmaf_grid) == 4 + 4 + 4 * 8 + 5 * 4 + 4 + 8


def test_validation_without_gpu(pkg):
    import gmaf_inputs as gi
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(3, 32)), 1) == 0          # INVALID_MESH
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(100, 80, "short")), 1) == 0  # too coarse
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(64, 32)), 0) == 0
    # row offsets are 32-bit in the iteration kernels: (n_y + 16) n_theta must stay below 2^31
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(65536, 32768 - 16)), 1) == 0
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(65536, 32768 - 17)), 1) > 0
    ctx = C.c_void_p()
    g = pkg.make_grid(gi.grid(64, 32))
    # a NULL workspace is rejected before any CUDA call
    code = pkg.lib().gmaf_create(C.byref(g), 1, None, None, 0, None, C.byref(ctx))
    assert code == -8


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle (the oracle is test infrastructure)."""
    src_dir = os.path.join(ROOT, "paper_2511_06824_b200")
    for dirpath, _, files in os.walk(src_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gmaf_oracle" not in txt, f


def test_row_slab_sizing_without_gpu(pkg):
    """GMAF_SHARD_ROWS_P2P: each rank stores its own rows + 4 halo rows per side of all K
    conditions (include/gmaf.h gmaf_slab); slabs thinner than 8 rows are rejected."""
    import gmaf_inputs as gi
    g = pkg.make_grid(gi.grid(2048, 1024, "short"))
    full = pkg.gmaf_workspace_bytes(g, 9)
    field = 2048 * 9 * 8                                   # one row of one field, all K
    sizes = []
    for r in range(4):
        d, _ = pkg.make_dist(r, 4, None, p2p=True, shard="rows")
        nb = pkg.gmaf_workspace_bytes(g, 9, d)
        stored = 256 + (4 if r > 0 else 0) + (4 if r < 3 else 0)
        assert 9 * field * stored <= nb <= 9 * field * stored + (64 << 20), (r, nb)
        sizes.append(nb)
    assert max(sizes) < full / 3
    d, _ = pkg.make_dist(0, 8, None, p2p=True, shard="rows")
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(64, 60)), 1, d) == 0      # 60 < 8 rows x 8
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(64, 64)), 1, d) > 0
    d, _ = pkg.make_dist(0, 9, None, p2p=True, shard="rows")
    assert pkg.gmaf_workspace_bytes(pkg.make_grid(gi.grid(64, 512)), 1, d) == 0     # > 8 ranks
