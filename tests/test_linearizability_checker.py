"""Pins of the per-key linearizability checker (tests/linearizability.py) used
for hive_mixed_concurrent: hand-made histories with a known answer, and a
brute force over every order of small random histories."""
import itertools

import numpy as np

from linearizability import check_batch, check_key


def test_hand_histories():
    A, P = (False, None), lambda v: (True, v)
    assert check_key(A, [(3, 7, 0)], [], [(False, None)], P(7)) == ["I"]          # find before the insert
    assert check_key(A, [(3, 7, 0)], [], [(True, 7)], P(7)) == ["I"]
    assert check_key(A, [(3, 7, 0)], [], [(True, 8)], P(7)) is None                # value never stored
    assert check_key(P(5), [], [], [(False, None)], P(5)) is None                 # present throughout
    assert check_key(P(5), [(1, 9, 1)], [(2, 1)], [(True, 9), (False, None)], A) == ["I", "E"]
    assert check_key(P(5), [(1, 9, 0)], [(2, 1)], [], P(9)) == ["E", "I"]         # erase, then re-insert
    assert check_key(P(5), [(1, 9, 1)], [(2, 1)], [], P(9)) is None               # status contradicts E, I
    # group members must agree, the value is the highest index's
    assert check_key(A, [(1, 4, 0), (6, 8, 1)], [], [], P(8)) is None
    assert check_key(A, [(1, 4, 0), (6, 8, 0)], [], [], P(8)) == ["I"]
    assert check_key(A, [(1, 4, 0), (6, 8, 0)], [], [], P(4)) is None


def _brute(s0, ins, era, finds, sf):
    """Every interleaving of the groups and finds, simulated op by op."""
    evs = ([("I",)] if ins else []) + ([("E",)] if era else []) + [("F", f, v) for f, v in finds]
    for perm in itertools.permutations(range(len(evs))):
        st, ok = s0, True
        for j in perm:
            e = evs[j]
            if e[0] == "I":
                stat = {s for _, _, s in ins}
                ok = len(stat) == 1 and stat.pop() == (1 if st[0] else 0)
                st = (True, max(ins)[1])
            elif e[0] == "E":
                stat = {s for _, s in era}
                ok = len(stat) == 1 and stat.pop() == (1 if st[0] else 0)
                st = (False, None)
            else:
                ok = (e[1] and st[0] and st[1] == e[2]) or (not e[1] and not st[0])
            if not ok:
                break
        if ok and st == sf:
            return True
    return False


def test_checker_equals_brute_force():
    rng = np.random.default_rng(3)
    for _ in range(3000):
        vals = [1, 2]
        s0 = (True, 1) if rng.random() < 0.5 else (False, None)
        ins = [(int(i), int(rng.choice(vals)), int(rng.integers(0, 2))) for i in range(int(rng.integers(0, 3)))]
        if ins and rng.random() < 0.7:                     # mostly consistent group statuses
            ins = [(i, v, ins[0][2]) for i, v, _ in ins]
        era = [(10 + i, int(rng.integers(0, 2))) for i in range(int(rng.integers(0, 2)))]
        finds = [(bool(rng.integers(0, 2)), int(rng.choice(vals))) for _ in range(int(rng.integers(0, 3)))]
        finds = [(f, v if f else None) for f, v in finds]
        sf = (True, int(rng.choice(vals))) if rng.random() < 0.5 else (False, None)
        assert (check_key(s0, ins, era, finds, sf) is not None) == _brute(s0, ins, era, finds, sf)


def test_batch_level_checks():
    before = {1: 10, 2: 20, 3: 30}
    ops = [1, 2, 0, 0, 3]
    keys = [1, 2, 3, 4, 5]
    vals = [11, 0, 0, 0, 0]
    after = {1: 11, 3: 30}
    assert check_batch(before, ops, keys, vals, [1, 1, 1, 0, 0], [0, 0, 30, 0, 0], after) == 4
    try:
        check_batch(before, ops, keys, vals, [1, 1, 1, 0, 0], [0, 0, 30, 0, 0], {1: 11, 3: 31})
        raise RuntimeError("missed a changed value")
    except AssertionError:
        pass
