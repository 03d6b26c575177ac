"""Drop-in `muxsim simulate`: the reference's config /
plan.json / trace.csv in, records.csv / metrics.json / poolstats.json out,
byte-identical to the unmodified reference CLI on the same inputs (goldens in
tests/golden/wire, made by make_wire_golden.sh with oracle/_ref/muxsim)."""
import json
import os

import pytest

from paper_2404_02015_b200 import muxsim_cli as simulate, wire

G = os.path.join(os.path.dirname(__file__), "golden", "wire")


@pytest.mark.parametrize("case", ["pair", "mesh", "b200prof", "empq"])
def test_priced_outputs_byte_identical_to_reference(case, tmp_path):
    out = tmp_path / "out"
    rc = simulate.main(["-c", os.path.join(G, f"cfg_{case}.json"), "-p", os.path.join(G, f"plan_{case}.json"),
                        "-t", os.path.join(G, f"trace_{case}.csv"), "-o", str(out)])
    assert rc == 0
    for name, golden in (("records.csv", f"records_{case}.csv"), ("metrics.json", f"metrics_{case}.json"),
                         ("poolstats.json", f"poolstats_{case}.json")):
        with open(out / name, "rb") as f, open(os.path.join(G, golden), "rb") as g:
            assert f.read() == g.read(), name


def test_nlohmann_number_format():
    # nlohmann::json dump: shortest round-trip digits, exponent form outside [1e-4, 1e15)
    cases = {0.0: "0.0", 2.0: "2.0", 0.1: "0.1", 1e-4: "0.0001", 1e-5: "1e-05", 1e15: "1e+15",
             1.5e15: "1.5e+15", 123456789.125: "123456789.125", -2.5e-7: "-2.5e-07", 1e22: "1e+22"}
    for x, want in cases.items():
        assert wire._dump(x) == want + "\n", x
    assert wire._dump({"a": [], "b": [1, 2.0], "c": "x"}) == '{\n  "a": [],\n  "b": [\n    1,\n    2.0\n  ],\n  "c": "x"\n}\n'


def test_percentile_nearest_rank():
    assert wire._percentile([3.0, 1.0, 2.0], 0.99) == 3.0
    assert wire._percentile(list(range(100)), 0.5) == 49


def test_trace_round_trip(tmp_path):
    exp = wire.load_config(os.path.join(G, "cfg_pair.json"))
    trace = wire.load_trace(os.path.join(G, "trace_pair.csv"), exp.names)
    p = tmp_path / "t.csv"
    wire.save_trace(str(p), trace, exp.names)
    with open(p, "rb") as f, open(os.path.join(G, "trace_pair.csv"), "rb") as g:
        assert f.read() == g.read()  # %.17g round trip (workload.cpp:138-149)


def test_config_errors_map_to_exit_code_1(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"cluster": {"num_nodes": 1, "gpus_per_node": 1, "gpu_memory_gb": 80}, '
                   '"llms": [{"name": "x", "model": "no-such-model"}]}')
    assert simulate.main(["-c", str(bad), "-p", os.path.join(G, "plan_pair.json"),
                          "-t", os.path.join(G, "trace_pair.csv"), "-o", str(tmp_path / "o")]) == 1
    missing = tmp_path / "t.csv"
    missing.write_text("id,llm,arrival_s,prompt_len,output_len\n0,nobody,0.5,3,4\n")
    assert simulate.main(["-c", os.path.join(G, "cfg_pair.json"), "-p", os.path.join(G, "plan_pair.json"),
                          "-t", str(missing), "-o", str(tmp_path / "o")]) == 1


def test_power_law_rates():
    assert wire.gen_rates(3, 1.0, 6.0) == [6.0, 3.0, 2.0]


def test_config_validation_matches_reference(tmp_path):
    """config.cpp:28-39 check_keys + range checks: typos and bad values are
    ConfigErrors (exit 1), as in the reference CLI."""
    base = {"cluster": {"num_nodes": 1, "gpus_per_node": 1, "gpu_memory_gb": 80},
            "llms": [{"name": "x", "model": "7b"}]}
    import copy
    import json as _json
    bad = []
    c = copy.deepcopy(base); c["sim"] = {"quota_low_mrk": 0.3}; bad.append(c)          # typo
    c = copy.deepcopy(base); c["sim"] = {"decode_sm": 1.5}; bad.append(c)              # range
    c = copy.deepcopy(base); c["sim"] = {"token_budget": 7.5}; bad.append(c)           # type
    c = copy.deepcopy(base); c["llms"][0]["prompt_len"] = {"kind": "empirical", "values": [1, 2],
                                                           "weights": [1]}; bad.append(c)
    c = copy.deepcopy(base); c["llms"].append({"name": "x", "model": "13b"}); bad.append(c)  # duplicate
    c = copy.deepcopy(base); c["profile"] = {"tp_efficiency": 0.2}; bad.append(c)
    for i, cfg in enumerate(bad):
        p = tmp_path / f"bad{i}.json"
        p.write_text(_json.dumps(cfg))
        with pytest.raises(wire.ConfigError):
            wire.load_config(str(p))
    ok = copy.deepcopy(base)
    ok["sim"] = {"quota_low_mark": 0.3, "quota_high_mark": 0.6, "quota_step_frac": 0.25}
    ok["llms"][0]["prompt_len"] = {"kind": "empirical", "values": [10, 100], "weights": [3, 1]}
    p = tmp_path / "ok.json"
    p.write_text(_json.dumps(ok))
    exp = wire.load_config(str(p))
    assert (exp.params.quota_low_mark, exp.params.quota_high_mark, exp.params.quota_step_frac) == (0.3, 0.6, 0.25)
    assert exp.entries[0].mean_prompt_tokens == (10 * 3 + 100 * 1) / 4  # weighted (workload.cpp:66-76)
    assert exp.entries[0].mean_output_tokens == 64.0                     # LlmConfig default (config.hpp:27)


def test_plan_split_and_unit_pools_match_reference():
    """cluster.split_plan routes each request to its model's unit
    (run_simulation, sim_engine.cpp:370-413) and unit_pool_blocks is
    UnitSim::pool_blocks (sim_engine.cpp:172-186): the reference CLI's
    poolstats total_blocks for the 2-unit tp=2 mesh golden."""
    import json as _json

    from paper_2404_02015_b200 import cluster
    exp = wire.load_config(os.path.join(G, "cfg_mesh.json"))
    placement = wire.load_plan(os.path.join(G, "plan_mesh.json"), exp.names)
    trace = wire.load_trace(os.path.join(G, "trace_mesh.csv"), exp.names)
    assert placement.gpu_ids == [[0, 1], [2, 3]]
    jobs = cluster.split_plan(exp.entries, trace, placement, exp.gpu_memory_bytes, exp.params, exp.profile,
                              "lockstep")
    assert [j.unit for j in jobs] == [0, 1] and [j.gpu_ids for j in jobs] == [[0, 1], [2, 3]]
    assert sorted(r.id for j in jobs for r in j.trace) == sorted(r.id for r in trace)
    for j in jobs:
        for r in j.trace:
            orig = next(t for t in trace if t.id == r.id)
            assert j.members[r.llm] == orig.llm
    with open(os.path.join(G, "poolstats_mesh.json")) as f:
        want = [u["total_blocks"] for u in _json.load(f)["units"]]
    got = [cluster.unit_pool_blocks([e.spec for e in j.entries], len(j.gpu_ids), exp.gpu_memory_bytes,
                                    exp.params.activation_reserve_frac) for j in jobs]
    assert got == want


def test_profile_tp_allreduce_keys(tmp_path):
    """B200 extension keys (wire.TP_KEYS): both or none, non-negative; they
    append after the reference's 7 (and the HBM form's 4) profile values."""
    from paper_2404_02015_b200 import wire
    base = json.load(open(os.path.join(G, "cfg_b200prof.json")))
    cfg = dict(base, profile=dict(base["profile"], allreduce_alpha_ms=0.02, allreduce_ms_per_mib=0.004))
    p = tmp_path / "c.json"
    p.write_text(json.dumps(cfg))
    exp = wire.load_config(str(p))
    assert len(exp.profile) == 9 and exp.profile[-2:] == [0.02, 0.004]
    cfg["profile"].pop("allreduce_ms_per_mib")
    p.write_text(json.dumps(cfg))
    with pytest.raises(wire.ConfigError):
        wire.load_config(str(p))
    cfg["profile"].update(allreduce_ms_per_mib=-1.0)
    p.write_text(json.dumps(cfg))
    with pytest.raises(wire.ConfigError):
        wire.load_config(str(p))
