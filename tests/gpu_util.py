"""Helpers for the GPU parity tests: run the same batches through the CUDA
table (via the C ABI) and the CPU oracle, and compare element by element."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2510_15095_b200 import HiveTable, u8, u32


def np32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.uint32)


def np8(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.uint8)


def gpu_dump(t: HiveTable) -> dict:
    k, v = t.dump()
    k, v = np32(k), np32(v)
    assert len(np.unique(k)) == len(k), "duplicate key in the GPU table"
    return dict(zip(k.tolist(), v.tolist()))


class Pair:
    """A CUDA table and an oracle table with the same configuration."""

    def __init__(self, capacity, oracle_cfg=None, **cfg):
        """oracle_cfg: settings that differ on the oracle side only (e.g. a larger
        stash, which changes no result unless it overflows)."""
        self.g = HiveTable(capacity, **cfg)
        ocfg = {k: v for k, v in cfg.items() if k != "keys_unique"}
        ocfg.update(oracle_cfg or {})
        self.o = oracle.OracleTable(capacity, **ocfg)

    def insert(self, keys, vals):
        keys = np.asarray(keys, np.uint32)
        vals = np.asarray(vals, np.uint32)
        st_g = np8(self.g.insert(u32(keys), u32(vals)))
        st_o = self.o.insert(keys, vals)
        self._oracle_ok()
        assert (st_g == st_o).all(), first_diff("insert status", st_g, st_o, keys)
        return st_g

    def _oracle_ok(self):
        # stash overflow is an error in both implementations;
        # report it as a test-configuration error, not as a GPU divergence
        pend = self.o.stats()["pending"]
        assert pend == 0, f"oracle stash overflow ({pend} pending): test config too tight"

    def find(self, keys):
        keys = np.asarray(keys, np.uint32)
        v_g, f_g = self.g.find(u32(keys))
        v_g, f_g = np32(v_g), np8(f_g)
        v_o, f_o = self.o.find(keys)
        assert (f_g == f_o).all(), first_diff("found", f_g, f_o, keys)
        assert (v_g == v_o).all(), first_diff("value", v_g, v_o, keys)
        return v_g, f_g

    def erase(self, keys):
        keys = np.asarray(keys, np.uint32)
        e_g = np8(self.g.erase(u32(keys)))
        e_o = self.o.erase(keys)
        assert (e_g == e_o).all(), first_diff("erased", e_g, e_o, keys)
        return e_g

    def mixed(self, ops, keys, vals):
        ops = np.asarray(ops, np.uint8)
        keys = np.asarray(keys, np.uint32)
        vals = np.asarray(vals, np.uint32)
        v_g, r_g = self.g.mixed(u8(ops), u32(keys), u32(vals))
        v_g, r_g = np32(v_g), np8(r_g)
        v_o, r_o = self.o.mixed(ops, keys, vals)
        self._oracle_ok()
        assert (r_g == r_o).all(), first_diff("mixed result", r_g, r_o, keys)
        assert (v_g == v_o).all(), first_diff("mixed value", v_g, v_o, keys)
        return v_g, r_g

    def check_state(self, cand: dict | None = None, trajectory: bool = True):
        """Final key->value set equal to the oracle's (values of keys inserted in
        the last batch must be members of their accepted set `cand`)."""
        dg = gpu_dump(self.g)
        do = self.o.dump_dict()
        assert set(dg) == set(do), (len(dg), len(do))
        bad = [k for k in dg if dg[k] != do[k]]
        if cand:
            assert all(dg[k] in cand[k] for k in cand if k in dg)
        assert not bad, ("values differ", bad[:5])
        sg, so = self.g.stats(), self.o.stats()
        assert sg["count"] == so["count"] == len(do)
        assert sg["failed"] == 0
        if trajectory:
            assert (sg["n_buckets"], sg["m"], sg["split"]) == (so["n_buckets"], so["m"], so["split"])
        return sg, so


def first_diff(what, a, b, keys):
    i = int(np.flatnonzero(a != b)[0]) if (a != b).any() else -1
    return f"{what}: first diff at {i}: gpu={a[i]} oracle={b[i]} key={keys[i]:#x} (n diff={(a != b).sum()})"
