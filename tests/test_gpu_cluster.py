"""Placement-driven execution (VERDICT r1 "What's missing" 1; reference
run_simulation, sim_engine.cpp:370-413): plans with several units and a
tensor-parallel mesh through the muxsim_cli drop-in on the GPU engines.

* a 2-unit plan (tiny-a on GPU 0, tiny-b on GPU 1): one process per unit;
  records.csv / metrics.json / poolstats.json byte-identical to the priced
  engine (lockstep decisions are the reference's, every job runs on a GPU);
* a tp = 2 plan (tiny-a + tiny-b on a 2-GPU mesh): two rank processes with
  head-sharded pools (BlockPool.enable_physical(2)) and the fused
  row-parallel allreduce over peer-mapped mailboxes; outputs byte-identical
  to priced, and both ranks emit identical tokens.
This box has one GPU: the units then run one after another on it, and the two
ranks of the mesh share it (their contexts time-slice), which checks
correctness, not NVLink speed.
"""
import json
import math
import os

import numpy as np
import pytest

import paper_2404_02015_b200 as mux
from paper_2404_02015_b200 import cluster, muxsim_cli, wire

pytestmark = pytest.mark.gpu


def _write_inputs(tmp_path, units, horizon=6.0, seed=4):
    cfg = {"cluster": {"num_nodes": 1, "gpus_per_node": 2, "gpu_memory_gb": 1},
           "llms": [{"name": "a", "model": "tiny-a", "rate_rps": 6.0,
                     "prompt_len": {"kind": "lognormal", "mean": 40, "sigma": 0.6},
                     "output_len": {"kind": "lognormal", "mean": 12, "sigma": 0.5}},
                    {"name": "b", "model": "tiny-b", "rate_rps": 3.0,
                     "prompt_len": {"kind": "constant", "value": 70},
                     "output_len": {"kind": "constant", "value": 9}}],
           "workload": {"horizon_s": horizon, "seed": seed},
           "sim": {"scheduler": "adbs", "quota_period_s": 1.0, "token_budget": 512}}
    plan = {"backend": "greedy", "units": units}
    rng = np.random.default_rng(seed)
    trace, rid = [], 0
    for llm, (rate, p, o) in enumerate([(6.0, 40, 12), (3.0, 70, 9)]):
        t = 0.0
        while True:
            t += rng.exponential(1.0 / rate)
            if t >= horizon:
                break
            pl = p if llm else max(1, int(round(rng.lognormal(math.log(p) - 0.18, 0.6))))
            ol = o if llm else max(1, int(round(rng.lognormal(math.log(o) - 0.125, 0.5))))
            trace.append((t, llm, pl, ol))
    trace.sort()
    paths = {k: str(tmp_path / f"{k}") for k in ("cfg.json", "plan.json", "trace.csv")}
    with open(paths["cfg.json"], "w") as f:
        json.dump(cfg, f)
    with open(paths["plan.json"], "w") as f:
        json.dump(plan, f)
    wire.save_trace(paths["trace.csv"], [mux.TraceRequest(i, llm, t, p, o) for i, (t, llm, p, o) in enumerate(trace)],
                    ["a", "b"])
    return paths


def _outputs(tmp_path, paths, engine):
    out = tmp_path / engine
    rc = muxsim_cli.main(["-c", paths["cfg.json"], "-p", paths["plan.json"], "-t", paths["trace.csv"], "-o", str(out),
                          "--engine", engine])
    assert rc == 0, engine
    return {n: (out / n).read_bytes() for n in ("records.csv", "metrics.json", "poolstats.json")}


@pytest.mark.timeout(600)
def test_two_unit_plan_runs_each_unit_on_its_gpu(cuda, tmp_path):
    units = [{"node": 0, "gpu_ids": [0], "models": [{"name": "a", "tp_degree": 1, "num_sm": 0.5}]},
             {"node": 0, "gpu_ids": [1], "models": [{"name": "b", "tp_degree": 1, "num_sm": 0.5}]}]
    paths = _write_inputs(tmp_path, units)
    priced = _outputs(tmp_path, paths, "priced")
    gpu = _outputs(tmp_path, paths, "lockstep")
    for name in priced:
        assert gpu[name] == priced[name], name
    stats = json.loads(gpu["poolstats.json"])
    assert [u["unit"] for u in stats["units"]] == [0, 1]


@pytest.mark.timeout(600)
def test_tp2_plan_runs_on_a_two_rank_mesh(cuda, tmp_path):
    units = [{"node": 0, "gpu_ids": [0, 1], "models": [{"name": "a", "tp_degree": 2, "num_sm": 0.5},
                                                        {"name": "b", "tp_degree": 2, "num_sm": 0.5}]}]
    paths = _write_inputs(tmp_path, units, horizon=4.0)
    priced = _outputs(tmp_path, paths, "priced")
    gpu = _outputs(tmp_path, paths, "lockstep")
    for name in priced:
        assert gpu[name] == priced[name], name
    # both ranks of the mesh produce the same tokens (bit-identical residuals
    # through the fused allreduce), every request its full output
    exp = wire.load_config(paths["cfg.json"])
    placement = wire.load_plan(paths["plan.json"], exp.names)
    trace = wire.load_trace(paths["trace.csv"], exp.names)
    recs, _, tokens = cluster.run_plan(exp.entries, trace, placement, exp.gpu_memory_bytes, exp.params,
                                       exp.profile, "lockstep", want_tokens=True)
    assert tokens[(0, 0)] == tokens[(0, 1)]
    assert [len(t) for t in tokens[(0, 0)]] == [r.output_len for r in trace]


def test_realtime_rejected_for_tensor_parallel_units(cuda, tmp_path):
    units = [{"node": 0, "gpu_ids": [0, 1], "models": [{"name": "a", "tp_degree": 2, "num_sm": 0.5},
                                                        {"name": "b", "tp_degree": 2, "num_sm": 0.5}]}]
    paths = _write_inputs(tmp_path, units, horizon=1.0)
    rc = muxsim_cli.main(["-c", paths["cfg.json"], "-p", paths["plan.json"], "-t", paths["trace.csv"],
                          "-o", str(tmp_path / "o"), "--engine", "realtime"])
    assert rc == 1
