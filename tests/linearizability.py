"""Per-key linearizability checker for hive_mixed_concurrent (test infrastructure).

Every op of one batch is concurrent with every other (they run in one kernel
launch), so real-time order adds no constraint: the batch is linearizable iff,
key by key (linearizability is local), SOME sequential order of that key's
operations explains every result and the key's final state.  Under the
contract of include/hive.h the state-changing operations of a key are at most
one insert group (all inserts of the key: one atomic step storing the value of
the highest-index insert; every member reports the presence before it) and one
erase group (all erases: one atomic step; every member reports the presence
before it); finds are atomic reads.  So each key has at most two state changes
and the orders to try are [], [I], [E], [I, E], [E, I]."""
from __future__ import annotations

from collections import defaultdict

import numpy as np

INVALID = 0xFFFFFFFF
OP_FIND, OP_INSERT, OP_ERASE = 0, 1, 2


def check_key(s0, ins, era, finds, sf):
    """s0 / sf: (present, value|None) before / after the batch.
    ins: list of (op index, value, status); era: list of (op index, status);
    finds: list of (found, value).  Returns the explaining order or None."""
    groups = {}
    if ins:
        st = {s for _, _, s in ins}
        if len(st) != 1:
            return None                          # members of one group must agree
        v = max(ins)[1]                          # highest op index's value
        groups["I"] = (st.pop(), v)
    if era:
        st = {s for _, s in era}
        if len(st) != 1:
            return None
        groups["E"] = (st.pop(), None)
    orders = [[]]
    if groups:
        names = sorted(groups)
        orders = [names] if len(names) == 1 else [names, names[::-1]]
    for order in orders:
        states = [s0]
        ok = True
        for g in order:
            status, v = groups[g]
            if status != (1 if states[-1][0] else 0):
                ok = False
                break
            states.append((True, v) if g == "I" else (False, None))
        if not ok or states[-1] != sf:
            continue
        if all(any((f and st[0] and st[1] == v) or (not f and not st[0]) for st in states) for f, v in finds):
            return order
    return None


def check_batch(before: dict, ops, keys, vals, result, vals_out, after: dict):
    """Raises AssertionError with the first violating key; returns the number
    of keys whose ops were checked."""
    ops, keys, vals = np.asarray(ops), np.asarray(keys, np.uint32), np.asarray(vals, np.uint32)
    result, vals_out = np.asarray(result), np.asarray(vals_out, np.uint32)
    per = defaultdict(lambda: ([], [], []))
    for i, (o, k) in enumerate(zip(ops.tolist(), keys.tolist())):
        if o > 2:
            assert result[i] == 0 and vals_out[i] == 0, ("invalid opcode result", i)
            continue
        if k == INVALID:
            assert result[i] == (2 if o == OP_INSERT else 0) and vals_out[i] == 0, ("reserved key", i)
            continue
        if o != OP_FIND:
            assert vals_out[i] == 0, ("vals_out of a non-find op", i)
        if o == OP_INSERT:
            per[k][0].append((i, int(vals[i]), int(result[i])))
        elif o == OP_ERASE:
            per[k][1].append((i, int(result[i])))
        else:
            assert result[i] in (0, 1), ("find result", i)
            per[k][2].append((bool(result[i]), int(vals_out[i]) if result[i] else None))
    for k, (ins, era, fnd) in per.items():
        s0 = (True, before[k]) if k in before else (False, None)
        sf = (True, after[k]) if k in after else (False, None)
        order = check_key(s0, ins, era, fnd, sf)
        assert order is not None, ("not linearizable", hex(k), s0, sf, ins[:4], era[:4], fnd[:4])
    untouched_before = {k: v for k, v in before.items() if k not in per}
    untouched_after = {k: v for k, v in after.items() if k not in per}
    assert untouched_before == untouched_after, "keys outside the batch changed"
    return len(per)
