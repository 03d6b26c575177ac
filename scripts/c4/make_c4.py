"""Config 4 (BASELINE.json configs[3]): a 7B/13B/30B/65B mix with power-law
popularity (alpha 0.9, max 4 rps; SURVEY.md Appendix B "Config-4
analogue") placed on a box of N B200s (179 GiB usable each) for N = 2, 4, 8:
2N models cycling 7b, 13b, 7b, 30b, 13b, 65b, 7b, 13b. Placement by the UNMODIFIED reference
planner (oracle/_ref/muxsim plan, greedy) restricted to tp_list [1] (every
model fits one 180 GB GPU; bench.py --placement runs one unit per rank) and
priced with the B200-measured profile. Run here (needs oracle/_ref); the
plans are committed data for bench.py --placement c4."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
MUXSIM = os.path.join(ROOT, "oracle", "_ref", "muxsim")
# 2 models per GPU in this order (the 65B first appears at 4 GPUs: with its KV
# it needs a GPU of its own)
CYCLE = ["7b", "13b", "7b", "30b", "13b", "65b", "7b", "13b"]


def config(n_gpus):
    llms = [{"name": f"m{i:02d}-{CYCLE[i % 8]}", "model": CYCLE[i % 8], "rate_rps": 1.0,
             "prompt_len": {"kind": "lognormal", "mean": 161, "sigma": 0.8},
             "output_len": {"kind": "lognormal", "mean": 338, "sigma": 0.8}} for i in range(2 * n_gpus)]
    return {"cluster": {"num_nodes": 1, "gpus_per_node": n_gpus, "gpu_memory_gb": 179},
            "llms": llms,
            "workload": {"horizon_s": 60, "seed": 4, "power_law": {"alpha": 0.9, "max_rate_rps": 4.0}},
            "placement": {"backend": "greedy", "tp_list": [1]},
            "sim": {"scheduler": "adbs"},
            "profile": json.load(open(os.path.join(ROOT, "profiles", "r01_b200_profile_7b.json")))["profile"]}


def main():
    for n in (2, 4, 8):
        cfg = os.path.join(HERE, f"cfg_g{n}.json")
        with open(cfg, "w") as f:
            json.dump(config(n), f, indent=1)
        plan = os.path.join(HERE, f"plan_g{n}.json")
        p = subprocess.run([MUXSIM, "plan", "-c", cfg, "-o", plan], capture_output=True, text=True)
        if p.returncode:
            sys.exit(f"muxsim plan g{n}: {p.stdout} {p.stderr}")
        units = json.load(open(plan))["units"]
        print(n, [[m["name"] for m in u["models"]] for u in units])


if __name__ == "__main__":
    main()
