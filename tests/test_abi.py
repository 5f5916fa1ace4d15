"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/tdvp.h declares, and its host-only schedule follows SURVEY.md App. A.
No compute calls (no GPU here)."""
import os
import re

import numpy as np
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


@pytest.mark.parametrize("L,p", [(2, 1), (9, 1), (8, 2), (12, 4), (16, 8), (10, 2), (100, 4), (64, 8)])
def test_plan1_protocol(L, p):
    """p1TDVP programs (tdvp_plan1, reading R-P1TDVP): (a) the message
    protocol of every segment and half is the p2TDVP one op for op (the NCCL
    and lane executors need nothing new); (b) per step every site is evolved
    forward by exactly dt and every bond that is not a segment boundary
    backward by exactly dt (time in units of dt/2: PAIR +1 per site, +2 when
    full; BACK -1; SITE_R/SITE_L +1 on the site unless skipped, -1 on the bond;
    FWD +2 when full else +1)."""
    comm = (3, 4, 5, 6)
    site = [0] * L
    bond = [0] * (L - 1)
    bounds = B.partition(L, p)
    boundary = {e for _, e in bounds[:-1]}
    for h in (1, 2):
        for q in range(p):
            p1, p2 = B.plan(L, p, h, q, one_site=True), B.plan(L, p, h, q)
            assert [op for op in p1 if op[0] in comm] == [op for op in p2 if op[0] in comm]
            for kind, j, full, build in p1:
                if kind == 1:
                    site[j] += 2 if full else 1
                    site[j + 1] += 2 if full else 1
                elif kind == 2:
                    site[j] -= 1
                elif kind == 7:
                    site[j] += 0 if full else 1
                    bond[j] -= 1
                elif kind == 8:
                    site[j] += 0 if full else 1
                    bond[j - 1] -= 1
                elif kind == 9:
                    site[j] += 2 if full else 1
    assert site == [2] * L
    assert all(bond[b] == -2 for b in range(L - 1) if b not in boundary), bond
    assert all(bond[b] == 0 for b in boundary)


def test_plan_serial_is_paper_sweep():
    # L->R pairs with backward singles, rightmost pair by the full dt
    L = 6
    h1 = B.plan(L, 1, 1, 0)
    assert h1 == [(1, 0, 0, 1), (2, 1, 0, 0), (1, 1, 0, 1), (2, 2, 0, 0), (1, 2, 0, 1), (2, 3, 0, 0),
                  (1, 3, 0, 1), (2, 4, 0, 0), (1, 4, 1, 2)]
    h2 = B.plan(L, 1, 2, 0)
    assert h2 == [(2, 4, 0, 0), (1, 3, 0, 2), (2, 3, 0, 0), (1, 2, 0, 2), (2, 2, 0, 0), (1, 1, 0, 2), (2, 1, 0, 0),
                  (1, 0, 0, 2)]


# ----------------------------------------------- N4 load-balanced partitions
def _brute_minmax(L, p, w):
    """Smallest achievable max segment cost over all contiguous partitions into
    p segments of >= 2 sites (exhaustive, small L)."""
    import itertools
    best = None
    for cuts in itertools.combinations(range(2, L - 1), p - 1):
        starts = (0,) + cuts
        ends = cuts + (L,)
        if any(b - a < 2 for a, b in zip(starts, ends)):
            continue
        v = max(sum(w[a:b]) for a, b in zip(starts, ends))
        best = v if best is None else min(best, v)
    return best


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("L,p", [(8, 2), (11, 4), (12, 2), (13, 4)])
def test_balanced_partition_is_optimal(L, p, seed):
    rng = np.random.default_rng(seed * 31 + L)
    chi = [1] + list(rng.integers(1, 40, size=L - 1)) + [1]
    w = [chi[j] * chi[j + 1] * (chi[j] + chi[j + 1]) for j in range(L)]
    b = B.balanced_partition(L, p, chi)
    assert len(b) == p and b[0][0] == 0 and b[-1][1] == L - 1
    assert all(b[q + 1][0] == b[q][1] + 1 for q in range(p - 1))
    assert all(e - s + 1 >= 2 for s, e in b)
    got = max(sum(w[s:e + 1]) for s, e in b)
    assert got == _brute_minmax(L, p, w)


def test_balanced_partition_saturated_profile():
    """Uniform chi: the balanced partition is the uniform one; a saturated
    profile (small chi at the chain ends) gives the edge segments more sites."""
    import tdvp_inputs as ti
    L = 64
    assert B.balanced_partition(L, 8, [1] + [16] * (L - 1) + [1])[1:-1] == B.partition(L, 8)[1:-1]
    chi = [1] + ti.saturated_chi_profile(L, 128) + [1]
    b = B.balanced_partition(L, 8, chi)
    sizes = [e - s + 1 for s, e in b]
    assert sizes[0] > 8 and sizes[-1] > 8
    w = [chi[j] * chi[j + 1] * (chi[j] + chi[j + 1]) for j in range(L)]
    cost = lambda bb: max(sum(w[s:e + 1]) for s, e in bb)  # noqa: E731
    assert cost(b) <= 0.875 * cost(B.partition(L, 8))  # 7 instead of 8 full-chi sites per segment


@pytest.mark.parametrize("L,p", [(8, 3), (8, 0), (5, 4)])
def test_balanced_partition_rejects_invalid(L, p):
    with pytest.raises(B.TdvpError):
        B.balanced_partition(L, p, [1] * (L + 1))


# ------------------------------------------ segment-lane channel protocol
SEND_R, RECV_L, SEND_L, RECV_R = 3, 4, 5, 6


@pytest.mark.parametrize("L,p", [(8, 2), (16, 4), (16, 8), (64, 8), (65, 8), (128, 16), (40, 20)])
def test_lane_channels_depth_one(L, p):
    """The concurrent-lane executor (engine.cu run_step_lanes) uses depth-1
    channels: per half-step every channel (q -> q+1 and q+1 -> q) carries at
    most one message and the neighbour receives it in the same half."""
    for h in (1, 2):
        progs = [B.plan(L, p, h, q) for q in range(p)]
        for q in range(p - 1):
            sr = sum(op[0] == SEND_R for op in progs[q])
            rl = sum(op[0] == RECV_L for op in progs[q + 1])
            sl = sum(op[0] == SEND_L for op in progs[q + 1])
            rr = sum(op[0] == RECV_R for op in progs[q])
            assert sr == rl <= 1 and sl == rr <= 1, (h, q, sr, rl, sl, rr)


@pytest.mark.parametrize("L,p", [(8, 2), (16, 4), (16, 8), (64, 8), (128, 16), (40, 20)])
def test_lane_execution_is_deadlock_free(L, p):
    """Simulate the lanes: p independent programs (half 1 then half 2, no
    barrier between halves), a SEND blocks while its depth-1 channel is full,
    a RECV while it is empty.  Under adversarial schedules (always advance the
    lowest- or highest-numbered runnable lane, or a seeded random one) every
    program completes."""
    import random
    progs = [B.plan(L, p, 1, q) + B.plan(L, p, 2, q) for q in range(p)]

    def chan(q, op):
        k = op[0]
        if k == SEND_R:
            return ("R", q)
        if k == RECV_L:
            return ("R", q - 1)
        if k == SEND_L:
            return ("L", q)
        if k == RECV_R:
            return ("L", q + 1)
        return None

    for policy in ("low", "high", "rand0", "rand1", "rand2"):
        rng = random.Random(policy)
        pc, full = [0] * p, {}
        while True:
            runnable = []
            for q in range(p):
                if pc[q] == len(progs[q]):
                    continue
                op = progs[q][pc[q]]
                c = chan(q, op)
                if c is None or (op[0] in (SEND_R, SEND_L) and not full.get(c)) or \
                        (op[0] in (RECV_L, RECV_R) and full.get(c)):
                    runnable.append(q)
            if not runnable:
                break
            q = runnable[0] if policy == "low" else runnable[-1] if policy == "high" else rng.choice(runnable)
            op = progs[q][pc[q]]
            c = chan(q, op)
            if c is not None:
                full[c] = op[0] in (SEND_R, SEND_L)
            pc[q] += 1
        assert all(pc[q] == len(progs[q]) for q in range(p)), (policy, pc)
        assert not any(full.values())
