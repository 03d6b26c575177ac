"""Restatement of the physical head-block id policy (TEST INFRASTRUCTURE).

Count semantics follow /root/reference/proj/src/kv_manager.cpp:74-140 (the
reference BlockPool only counts blocks, kv_manager.hpp:88-104). The physical
policy is this repo's own (csrc/host/kv.cpp) and is pinned here:
  * one LIFO free stack of ids, initially popping 0, 1, 2, ...;
  * a request's new 16-token row pops 2*L*H ids, assigned in
    (layer, head, K/V) order;
  * row records and device slots are recycled LIFO;
  * free pushes ids back in exact reverse pop order.
Pure Python; for small cases only.
"""
from __future__ import annotations


class PhysicalPoolRef:
    def __init__(self, total_blocks: int):
        self.total = total_blocks
        self.free_ids = list(range(total_blocks - 1, -1, -1))  # pop() -> 0 first
        self.models = {}

    def register(self, llm: int, layers: int, heads: int, block_tokens: int = 16):
        self.models[llm] = {"w": 2 * layers * heads, "bt": block_tokens, "reqs": {},
                            "free_rec": [], "n_rec": 0, "free_slot": [], "n_slot": 0}

    def rows_for(self, llm, tokens):
        bt = self.models[llm]["bt"]
        return (tokens + bt - 1) // bt

    def grow(self, llm: int, rid: int, tokens_after: int):
        m = self.models[llm]
        r = m["reqs"].setdefault(rid, {"rows": [], "slot": -1, "tokens": 0})
        need = self.rows_for(llm, tokens_after) - len(r["rows"])
        if need > 0 and r["slot"] < 0:
            if m["free_slot"]:
                r["slot"] = m["free_slot"].pop()
            else:
                r["slot"] = m["n_slot"]
                m["n_slot"] += 1
        for _ in range(need):
            if m["free_rec"]:
                rec = m["free_rec"].pop()
            else:
                rec = m["n_rec"]
                m["n_rec"] += 1
            ids = [self.free_ids.pop() for _ in range(m["w"])]
            r["rows"].append((rec, ids))
        r["tokens"] = tokens_after

    def free(self, llm: int, rid: int):
        m = self.models[llm]
        r = m["reqs"].pop(rid)
        for rec, ids in reversed(r["rows"]):
            self.free_ids.extend(reversed(ids))
            m["free_rec"].append(rec)
        if r["slot"] >= 0:
            m["free_slot"].append(r["slot"])

    def block_table(self, llm: int, rid: int) -> list[int]:
        r = self.models[llm]["reqs"].get(rid)
        return [i for _, ids in r["rows"] for i in ids] if r else []

    def slot(self, llm: int, rid: int) -> int:
        r = self.models[llm]["reqs"].get(rid)
        return r["slot"] if r else -1
