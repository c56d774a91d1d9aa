"""Brute-force PHASED dictionary model (SURVEY §8(c) "Batch semantics
contract") — a plain Python dict, used to pin the oracle and to check the GPU.

A batch applies all INSERT ops, then all ERASE ops, then all FIND ops.
* insert status = present(k) at INSERT-phase start (2 = reserved key);
  the final value is one of the values inserted for k in the batch
  (``cand`` records the accepted set; last-write-wins is one member).
* erase output = present(k) at ERASE-phase start.
* find output  = (present, value) at FIND-phase start.
"""
from __future__ import annotations

import numpy as np

INVALID = 0xFFFFFFFF
OP_FIND, OP_INSERT, OP_ERASE = 0, 1, 2


class PhasedModel:
    def __init__(self):
        self.d: dict[int, int] = {}

    def insert(self, keys, vals):
        keys = [int(k) for k in keys]
        vals = [int(v) for v in vals]
        start = self.d
        status = np.zeros(len(keys), np.uint8)
        cand: dict[int, set] = {}
        new = dict(start)
        for i, (k, v) in enumerate(zip(keys, vals)):
            if k == INVALID:
                status[i] = 2
                continue
            status[i] = 1 if k in start else 0
            cand.setdefault(k, set()).add(v)
            new[k] = v                      # last write wins (one accepted member)
        self.d = new
        return status, cand

    def erase(self, keys):
        keys = [int(k) for k in keys]
        start = self.d
        out = np.array([1 if (k != INVALID and k in start) else 0 for k in keys], np.uint8)
        self.d = {k: v for k, v in start.items() if k not in set(keys)}
        return out

    def find(self, keys):
        keys = [int(k) for k in keys]
        found = np.array([1 if k in self.d else 0 for k in keys], np.uint8)
        vals = np.array([self.d.get(k, 0) for k in keys], np.uint32)
        return vals, found

    def mixed(self, ops, keys, vals):
        ops = np.asarray(ops)
        keys = np.asarray(keys, np.uint32)
        vals = np.asarray(vals, np.uint32)
        n = len(keys)
        res = np.zeros(n, np.uint8)
        vo = np.zeros(n, np.uint32)
        ii = np.flatnonzero(ops == OP_INSERT)
        ee = np.flatnonzero(ops == OP_ERASE)
        ff = np.flatnonzero(ops == OP_FIND)
        cand = {}
        if len(ii):
            st, cand = self.insert(keys[ii], vals[ii])
            res[ii] = st
        if len(ee):
            res[ee] = self.erase(keys[ee])
        if len(ff):
            v, f = self.find(keys[ff])
            res[ff] = f
            vo[ff] = v
        return vo, res, cand


def accept_values(model_d: dict, got_d: dict, cand: dict):
    """Any-value rule: keys inserted in the batch may hold any candidate value;
    every other key must match exactly.  Returns the list of violations."""
    bad = []
    if set(model_d) != set(got_d):
        missing = set(model_d) - set(got_d)
        extra = set(got_d) - set(model_d)
        bad.append(("keyset", len(missing), len(extra)))
        return bad
    for k, v in got_d.items():
        if k in cand:
            if v not in cand[k]:
                bad.append(("value-not-candidate", k, v))
        elif model_d[k] != v:
            bad.append(("value", k, v, model_d[k]))
    return bad
