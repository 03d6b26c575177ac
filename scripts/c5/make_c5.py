"""Config 5 (BASELINE.json configs[4]): the 19-LLM endpoint mix (LLaMA
7B-65B, Table 1 of the paper: 65B x1, 30B x2, 13B x4, 7B x12; model of rank i
= MIX[(i * 7) % 19]) on 1 x 8 B200 (179 GiB usable per
GPU), power-law popularity (alpha 0.9) at four arrival-rate levels
(max_rate_rps 5 / 10 / 20 / 40), ShareGPT lengths. Placement from the
UNMODIFIED reference planner (oracle/_ref/muxsim plan, greedy, tp_list [1]:
every model fits one 180 GB GPU, and the real-time engine runs tp = 1 units),
traces from `muxsim gen-workload`, priced with the B200-measured profile
(profiles/r01_b200_profile_7b.json). Run here (needs oracle/_ref); the outputs
are committed data for scripts/slo_sweep_c5.sh."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
MUXSIM = os.path.join(ROOT, "oracle", "_ref", "muxsim")
MIX = ["65b"] + ["30b"] * 2 + ["13b"] * 4 + ["7b"] * 12
RATES = [5, 10, 20, 40]


def config(max_rate):
    llms = []
    for i in range(19):
        m = MIX[(i * 7) % 19]
        llms.append({"name": f"ep{i:02d}-{m}", "model": m, "rate_rps": 1.0,
                     "prompt_len": {"kind": "lognormal", "mean": 161, "sigma": 0.8},
                     "output_len": {"kind": "lognormal", "mean": 338, "sigma": 0.8}})
    return {"cluster": {"num_nodes": 1, "gpus_per_node": 8, "gpu_memory_gb": 179},
            "llms": llms,
            "workload": {"horizon_s": 20, "seed": 3, "power_law": {"alpha": 0.9, "max_rate_rps": max_rate}},
            "placement": {"backend": "greedy", "tp_list": [1]},
            "sim": {"scheduler": "adbs", "quota_period_s": 2.0, "warmup_s": 0.0},
            "metrics": {"slo_scales": [2, 4, 8, 16, 32]},
            # the B200-measured LatencyProfile (calibrate.py, reference form)
            "profile": json.load(open(os.path.join(ROOT, "profiles", "r01_b200_profile_7b.json")))["profile"]}


def main():
    for r in RATES:
        cfg = os.path.join(HERE, f"cfg_r{r}.json")
        with open(cfg, "w") as f:
            json.dump(config(r), f, indent=1)
        for cmd in (["plan", "-c", cfg, "-o", os.path.join(HERE, f"plan_r{r}.json")],
                    ["gen-workload", "-c", cfg, "-o", os.path.join(HERE, f"trace_r{r}.csv")]):
            p = subprocess.run([MUXSIM] + cmd, capture_output=True, text=True)
            if p.returncode:
                sys.exit(f"muxsim {cmd[0]} r{r}: {p.stdout} {p.stderr}")
        plan = json.load(open(os.path.join(HERE, f"plan_r{r}.json")))
        print(r, [[m["name"] for m in u["models"]] for u in plan["units"]])


if __name__ == "__main__":
    main()
