"""bench.py --placement: the committed config-4 placements (scripts/c4, made
by the unmodified reference planner) map one unit per rank, cover every
model of the config exactly once, and use only realizable tp = 1 units."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_plans_cover_the_config(world):
    units = bench.placement_plan("c4", world)
    assert len(units) == world
    cfg = json.load(open(os.path.join(ROOT, "scripts", "c4", f"cfg_g{world}.json")))
    assert sorted(m for u in units for m in u) == sorted(e["model"] for e in cfg["llms"])
    for u in units:  # every unit's weights fit one 180 GiB B200 with the 10% reserve
        assert sum(bench.WEIGHT_BYTES[m] for m in u) < 0.9 * bench.MESH_BYTES


def test_unit_models_default_is_one_copy_per_rank():
    class A:
        placement = ""
        models = "7b,13b"
    assert bench.unit_models(A, 1, 4) == ["7b", "13b"]
    A.placement = "c4"
    assert bench.unit_models(A, 1, 2) == bench.placement_plan("c4", 2)[1]
    assert bench.unit_models(A, 0, 1) == ["7b", "13b"]  # N = 1 is always the headline cfg2 unit


@pytest.mark.gpu
def test_bench_placement_two_ranks_on_one_gpu(tmp_path):
    """The N > 1 placement path end to end: 2 ranks (gloo, sharing the one
    GPU) each run their unit of plan_g2 and rank 0 prints the sums."""
    env = dict(os.environ, MUX_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--placement", "c4", "--batch", "8", "--e2e-steps", "2", "--attn-steps", "1"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert [u["models"] for u in line["run"]["units"]] == bench.placement_plan("c4", 2)
    assert line["config"]["units"] == [",".join(u) for u in bench.placement_plan("c4", 2)]


@pytest.mark.parametrize("rate", [5, 10, 20, 40])
def test_c5_sweep_inputs_are_consistent(rate):
    """scripts/c5 (config 5, 19 LLMs): every model placed exactly once on a
    tp = 1 unit that fits one GPU, and every trace row names a config model."""
    from paper_2404_02015_b200 import wire
    d = os.path.join(ROOT, "scripts", "c5")
    exp = wire.load_config(os.path.join(d, f"cfg_r{rate}.json"))
    plan = json.load(open(os.path.join(d, f"plan_r{rate}.json")))
    placed = [m["name"] for u in plan["units"] for m in u["models"]]
    assert sorted(placed) == sorted(exp.names) and len(exp.names) == 19
    for u in plan["units"]:  # empty meshes may be wider: they idle
        assert not u["models"] or (len(u["gpu_ids"]) == 1 and all(m["tp_degree"] == 1 for m in u["models"]))
    trace = wire.load_trace(os.path.join(d, f"trace_r{rate}.csv"), exp.names)
    assert trace and all(0 <= r.llm < 19 for r in trace)
