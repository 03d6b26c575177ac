"""`muxsim simulate` drop-in:

    python -m paper_2404_02015_b200.muxsim_cli -c cfg.json -p plan.json -t trace.csv -o out/ \\
        [--engine priced|lockstep|measured|realtime]

Reads the reference's config / plan.json / trace.csv and writes records.csv,
metrics.json and poolstats.json in the reference's formats
(/root/reference/proj/src/commands.cpp:265-298, 74-121; metrics.cpp:40-167).
Engines:
  priced    the reference's event loop and pricing model in libmux.so
            (CPU; records byte-identical to `muxsim simulate`)
  lockstep  the same decisions, every job executed on this GPU (random-init
            weights, synthetic prompt tokens); records identical to priced
  measured  job completions at measured device time (real serving latencies)
  realtime  jobs overlap across passes, completions when their device events
            fire (mux_unit_run_realtime; concurrency and contention measured)
The GPU engines run any plan: every unit on its own GPU mesh, one process
per tensor-parallel rank (cluster.run_plan; tp > 1 units in lockstep mode).
A box with fewer GPUs than the plan names runs the units one after another.
Exit codes follow the reference CLI (muxsim.cpp:51-63): 1 config error,
2 infeasible, 3 anything else.
"""
from __future__ import annotations

import argparse
import os
import sys

from . import cluster, wire
from ._lib import Infeasible, InvalidArgument
from .host import Unit, simulate


def _run_single(exp, placement, trace, engine):
    """A one-GPU plan, in this process."""
    specs = [exp.entries[i].spec for i in placement.members[0]]
    logical = cluster.unit_pool_blocks(specs, 1, exp.gpu_memory_bytes, exp.params.activation_reserve_frac)
    longest = max((r.prompt_len + r.output_len for r in trace), default=16)
    unit = Unit(specs, pool_blocks=logical, device_pool_blocks=logical, max_batch=512,
                max_prefill_tokens=max(exp.params.token_budget, longest), max_ctx=longest + 16,
                max_slots=len(trace) + 8, init_seed=1, init_std=0.02, partitions=len(specs) + 1)
    try:
        recs, _ = unit.run_lockstep([exp.entries[i] for i in placement.members[0]], trace,
                                    exp.gpu_memory_bytes, exp.params, profile=exp.profile,
                                    measured=engine == "measured", realtime=engine == "realtime")
        units = unit.last_stats()
        mem = placement.members[0]  # unit-local entry index -> config entry index
        for u in units:
            for m in u.llms:
                m.llm = mem[m.llm]
            u.samples = [(t, mem[li], used, q) for t, li, used, q in u.samples]
    finally:
        unit.close()
    return recs, units


def run(cfg_path: str, plan_path: str, trace_path: str, out_dir: str, engine: str = "priced") -> list:
    exp = wire.load_config(cfg_path)
    placement = wire.load_plan(plan_path, exp.names)
    trace = wire.load_trace(trace_path, exp.names)
    if engine == "priced":
        recs, units = simulate(exp.entries, trace, placement, exp.gpu_memory_bytes, exp.params, exp.profile,
                               stats=True)
    else:
        if exp.params.block_tokens != 16:
            raise wire.ConfigError("GPU engines: sim.block_tokens must be 16 (the kernels' 4 KiB head-blocks)")
        if len(placement.mesh_sizes) == 1 and placement.mesh_sizes[0] == 1:
            recs, units = _run_single(exp, placement, trace, engine)
        else:  # every unit on its own GPU mesh, one process per rank (cluster.run_plan)
            try:
                recs, units, _ = cluster.run_plan(exp.entries, trace, placement, exp.gpu_memory_bytes, exp.params,
                                                  exp.profile, engine)
            except ValueError as e:
                raise wire.ConfigError(str(e)) from None
    report = wire.compute_metrics(recs, exp, placement)
    os.makedirs(out_dir, exist_ok=True)
    wire.write_records_csv(os.path.join(out_dir, "records.csv"), recs, exp.names)
    with open(os.path.join(out_dir, "metrics.json"), "w") as f:
        f.write(wire.metrics_json(report, exp, units))
    with open(os.path.join(out_dir, "poolstats.json"), "w") as f:
        f.write(wire.poolstats_json(units, exp.names))
    return recs


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="simulate", description=__doc__.split("\n")[0])
    ap.add_argument("-c", "--config", required=True)
    ap.add_argument("-p", "--plan", required=True)
    ap.add_argument("-t", "--trace", required=True)
    ap.add_argument("-o", "--output", default="out")
    ap.add_argument("--engine", choices=["priced", "lockstep", "measured", "realtime"], default="priced")
    a = ap.parse_args(argv)
    try:
        recs = run(a.config, a.plan, a.trace, a.output, a.engine)
    except (wire.ConfigError, InvalidArgument) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except Infeasible as e:
        print(f"infeasible: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - the reference maps everything else to 3
        print(f"error: {e}", file=sys.stderr)
        return 3
    print(f"engine {a.engine}: {len(recs)} requests; wrote {a.output}/records.csv, metrics.json, poolstats.json")
    return 0


if __name__ == "__main__":
    sys.exit(main())
