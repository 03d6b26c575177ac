"""Drop-in `muxsim simulate`: the reference's config /
plan.json / trace.csv in, records.csv out, byte-identical to the unmodified
reference CLI on the same inputs (goldens in tests/golden/wire, made by
make_wire_golden.sh with oracle/_ref/muxsim)."""
import os

import pytest

from paper_2404_02015_b200 import muxsim_cli as simulate, wire

G = os.path.join(os.path.dirname(__file__), "golden", "wire")


@pytest.mark.parametrize("case", ["pair", "mesh"])
def test_priced_records_csv_byte_identical_to_reference(case, tmp_path):
    out = tmp_path / "out"
    rc = simulate.main(["-c", os.path.join(G, f"cfg_{case}.json"), "-p", os.path.join(G, f"plan_{case}.json"),
                        "-t", os.path.join(G, f"trace_{case}.csv"), "-o", str(out)])
    assert rc == 0
    with open(out / "records.csv", "rb") as f, open(os.path.join(G, f"records_{case}.csv"), "rb") as g:
        assert f.read() == g.read()


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
