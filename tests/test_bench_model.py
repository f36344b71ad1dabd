"""Host logic of bench.py (no GPU): the byte model the roofline line divides by.

The streamed kernels' algorithmic bytes per dof follow the store they read
("a compressed store must use that store's own byte model"):
the per-cell store's figures (u, b, D, U, H0-H2 in, u' out = 64 B/dof for a
sweep, ...), less 12 B/dof where the edge-deduplicated couplings are read and
8 B/dof where D is re-formed from the streamed couplings (DESIGN 7.5, 7.7)."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_canonical_per_cell_store(bench):
    # apply 56, sweep 64, zero-guess sweep 32, residual + restriction 58
    b = bench.BYTES_PER_DOF
    assert (b["apply"], b["sweep"], b["sweep_zero"], b["resid_restrict"]) == (56.0, 64.0, 32.0, 58.0)
    assert b["sweep_prolong"] == 64.0 + 2.0      # + a quarter of u_c per fine dof
    assert b["apply_pupdate"] == 56.0 + 16.0     # + z in, p_new out


def test_store_bytes_edge_store_level(bench):
    s = bench.store_bytes({"sweep": True, "apply": True, "resid_restrict": True})
    assert s["sweep"] == 44.0 and s["sweep_prolong"] == 46.0 and s["apply"] == 36.0
    assert s["apply_pupdate"] == 60.0             # streams D (DESIGN 7.1a)
    assert s["resid_restrict"] == 38.0 and s["sweep_zero"] == 32.0


def test_store_bytes_per_cell_level(bench):
    s = bench.store_bytes({"sweep": False, "apply": False, "resid_restrict": False})
    assert s["sweep"] == 56.0 and s["sweep_prolong"] == 58.0 and s["apply"] == 48.0
    assert s["apply_pupdate"] == 72.0
    assert s["resid_restrict"] == 58.0            # thread-per-column k_resid_restrict reads D
