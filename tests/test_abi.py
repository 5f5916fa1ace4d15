"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/tdvp.h declares, and its host-only schedule follows SURVEY.md App. A.
No compute calls (no GPU here)."""
import os
import re

import pytest

from paper_1912_06127_b200 import tdvp as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tdvp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tdvp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = B.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in B._SIGS, f"binding lacks {s}"


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(B.TdvpError) as e:
        B.Tdvp(4, 2, 5, 8)
    assert e.value.code == -4


@pytest.mark.parametrize("L,p", [(8, 1), (8, 2), (12, 4), (16, 8), (10, 2), (131, 8), (64, 2), (256, 8)])
def test_partition_matches_oracle(L, p):
    from oracle import plan_partition
    assert B.partition(L, p) == plan_partition(L, p)


@pytest.mark.parametrize("L,p", [(8, 3), (8, 0), (8, 6), (5, 4)])
def test_partition_rejects_invalid(L, p):
    with pytest.raises(B.TdvpError) as e:
        B.partition(L, p)
    assert e.value.code == -3


@pytest.mark.parametrize("L,p", [(2, 1), (9, 1), (8, 2), (12, 4), (16, 8), (10, 2), (100, 4), (64, 8)])
def test_plan_counts_and_messages(L, p):
    """Per half: N-1 forward pairs (full-dt pairs count twice) and N-2 backward
    singles (AMB-1 invariant, checked by P11); every bond gets total forward
    time dt; every send has a matching receive in the same order."""
    halves = {h: [B.plan(L, p, h, q) for q in range(p)] for h in (1, 2)}
    per_bond = [0.0] * (L - 1)
    n_fwd = 0
    for h in (1, 2):
        ops = [op for prog in halves[h] for op in prog]
        pairs = [op for op in ops if op[0] == 1]
        backs = [op for op in ops if op[0] == 2]
        n_fwd += len(pairs) + sum(op[2] for op in pairs)
        assert len(backs) == L - 2
        for op in pairs:
            per_bond[op[1]] += 1.0 if op[2] else 0.5
        # message matching between neighbours
        for q in range(p - 1):
            sends_r = [op for op in halves[h][q] if op[0] == 3]
            recvs_l = [op for op in halves[h][q + 1] if op[0] == 4]
            sends_l = [op for op in halves[h][q + 1] if op[0] == 5]
            recvs_r = [op for op in halves[h][q] if op[0] == 6]
            assert len(sends_r) == len(recvs_l)
            assert len(sends_l) == len(recvs_r)
    assert per_bond == [1.0] * (L - 1)
    assert n_fwd == 2 * (L - 1)


def test_plan_serial_is_paper_sweep():
    # L->R pairs with backward singles, rightmost pair by the full dt
    L = 6
    h1 = B.plan(L, 1, 1, 0)
    assert h1 == [(1, 0, 0, 1), (2, 1, 0, 0), (1, 1, 0, 1), (2, 2, 0, 0), (1, 2, 0, 1), (2, 3, 0, 0),
                  (1, 3, 0, 1), (2, 4, 0, 0), (1, 4, 1, 2)]
    h2 = B.plan(L, 1, 2, 0)
    assert h2 == [(2, 4, 0, 0), (1, 3, 0, 2), (2, 3, 0, 0), (1, 2, 0, 2), (2, 2, 0, 0), (1, 1, 0, 2), (2, 1, 0, 0),
                  (1, 0, 0, 2)]
