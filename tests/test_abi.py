"""CPU checks of the boundary: the C-ABI library builds, loads without a GPU and exports
every function include/bubblespec.h declares; host-only entry points work on CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bubblespec.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2605_08862_b200 import build

    path = build.build()
    return ctypes.CDLL(path)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bsx?_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["bs_draft_pool_put", "bs_draft_lookup", "bs_verify_step", "bs_commit",
              "bs_draft_pool_seal", "bs_draft_exchange", "bs_create", "bs_destroy"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_signatures_cover_header(lib):
    from paper_2605_08862_b200._lib import SIGNATURES

    assert set(declared_functions()) == set(SIGNATURES)


def test_create_without_gpu_fails_cleanly(lib):
    """No GPU here: bs_create must return BS_ERR_CUDA (3), never crash."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_08862_b200 import BubbleSpecError, Context

    with pytest.raises(BubbleSpecError) as e:
        Context(vocab=1024, device=0)
    assert e.value.status == 3


def test_invalid_config_rejected_before_device(lib):
    from paper_2605_08862_b200._lib import bs_config, load

    L = load()
    h = ctypes.c_void_p()
    cfg = bs_config(0, -1, 4, 32, 1, 4, 16, 4, 0, 0)
    assert L.bs_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    assert b"vocab" in L.bs_last_error(None)
    cfg = bs_config(1024, -1, 40, 32, 1, 4, 16, 4, 0, 0)
    assert L.bs_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    # the verify launch packs rollout counts into 21-bit fields
    cfg = bs_config(1024, -1, 4, 32, 1, 1 << 21, 16, 4, 0, 0)
    assert L.bs_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    assert b"max_rollouts" in L.bs_last_error(None)
    cfg = bs_config(600000, -1, 4, 32, 1, 4, 16, 4, 0, 0)
    assert L.bs_create(ctypes.byref(cfg), ctypes.byref(h)) == 1
    assert b"vocab" in L.bs_last_error(None)


def test_version_string(lib):
    from paper_2605_08862_b200._lib import load

    assert b"sm_100a" in load().bs_version()


def test_route_plan_host_logic():
    """bs_route_plan (the host half of bs_draft_exchange): owner = prompt mod world."""
    from paper_2605_08862_b200 import bs_route_plan

    world, max_seqs, max_tok = 3, 4, 20
    counts = np.array([2, 5, 3, 9, 0, 0], np.int64)
    offs = np.zeros((world, max_seqs + 1), np.int64)
    offs[0, :3] = [0, 2, 5]
    offs[1, :4] = [0, 4, 4, 9]
    prm = np.zeros((world, max_seqs), np.int32)
    prm[0, :2] = [3, 4]
    prm[1, :3] = [6, 1, 9]
    for rank in range(world):
        src, dst, ln, pr, nt = bs_route_plan(world, rank, counts, offs.ravel(), prm.ravel(),
                                             max_seqs, max_tok)
        assert all(p % world == rank for p in pr)
        assert nt == int(ln.sum())
        assert list(dst) == list(np.cumsum(ln) - ln)
    src, dst, ln, pr, nt = bs_route_plan(world, 0, counts, offs.ravel(), prm.ravel(), max_seqs,
                                         max_tok)
    assert list(pr) == [3, 6, 9] and list(ln) == [2, 4, 5] and list(src) == [0, 20, 24]


def _golden(tag):
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")):
        if line.startswith("# " + tag):
            return line
    raise KeyError(tag)


def test_metrics_from_counters_spec_hand_trace():
    """SPEC S:494-496 hand trace (tests/golden/spec_examples.txt 'metrics'): three verification
    steps emitting (2, 3, 1) tokens for (4, 4, 2) proposed drafts -> AL 2.0, DL 10/3, AR 0.3,
    through the engine's counter -> metric conversion (summarize_stats)."""
    import re

    from paper_2605_08862_b200.engine import summarize_stats

    line = _golden("metrics")
    emitted = [int(x) for x in re.search(r"emitted \(([\d,]+)\)", line).group(1).split(",")]
    proposed = [int(x) for x in re.search(r"proposed \(([\d,]+)\)", line).group(1).split(",")]
    al, num, den, ar = re.search(r"AL ([\d.]+), DL (\d+)/(\d+), AR ([\d.]+)", line).groups()
    st = np.zeros(41, dtype=np.uint64)
    st[0] = len(emitted)                          # verification steps
    st[2] = sum(emitted)                          # tokens they emitted
    st[4] = sum(e - 1 for e in emitted)           # accepted drafts (each step ends in a sample)
    st[5] = sum(proposed)
    for e in emitted:
        st[8 + e] += 1
    m = summarize_stats(st)
    assert m["acceptance_length"] == float(al)
    assert m["draft_length"] == int(num) / int(den)
    assert abs(m["acceptance_rate"] - float(ar)) < 1e-12
    assert m["streak_hist"][1:4] == [1, 1, 1]


def test_metric_identity_table1():
    """AR = (AL - 1) / DL (SURVEY c.6 metrics pin) on the paper's Table 1 rows (P:269, P:273,
    P:277, golden 'table1'): summarize_stats on counters built from each row's AL and DL
    reproduces the printed AR to the table's rounding."""
    import re

    from paper_2605_08862_b200.engine import summarize_stats

    line = _golden("table1")
    rows = re.findall(r"\(AL ([\d.]+), DL ([\d.]+), AR ([\d.]+)%\)|\(([\d.]+), ([\d.]+), ([\d.]+)%\)", line)
    assert len(rows) == 3
    for r in rows:
        al, dl, ar = [float(x) for x in (r[:3] if r[0] else r[3:])]
        steps = 10_000
        st = np.zeros(41, dtype=np.uint64)
        st[0] = steps
        st[2] = round(al * steps)
        st[4] = round((al - 1) * steps)
        st[5] = round(dl * steps)
        m = summarize_stats(st)
        assert abs(100 * m["acceptance_rate"] - ar) < 0.06, (al, dl, ar, m["acceptance_rate"])


def test_pool_sequences_from_pregen():
    """Pre-generated responses -> pool sequences (reading L4: [last M prompt tokens] +
    response, padding dropped, empty responses skipped), host logic of f1."""
    from paper_2605_08862_b200.pregen import pool_sequences

    tails = np.array([[-1, -1, 5, 6], [1, 2, 3, 4], [-1, 9, 9, 9]], dtype=np.int32)
    resp = np.array([[10, 11, 12, -1], [20, -1, -1, -1], [30, 31, 32, 33]], dtype=np.int32)
    sp, off, tok = pool_sequences([7, 8, 9], tails, resp, [3, 0, 4], M=3)
    assert list(sp) == [7, 9]
    assert list(off) == [0, 5, 12]
    assert list(tok) == [5, 6, 10, 11, 12, 9, 9, 9, 30, 31, 32, 33]
