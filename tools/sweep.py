"""Run bench.py over every workload (one B200) and summarise.

  python tools/sweep.py [--out gpurun_out/sweep] [--steps 5] [--workloads a,b,...]

Writes <out>/sweep_<workload>.json (the bench line) and <out>/summary.json.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALL = ["cfg3-rmc2", "cfg3-rmc3", "cfg1-rmc1", "cfg5-din", "cfg5-dien", "ncf", "wnd", "mt-wnd",
       "rmc1", "rmc2", "rmc3"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep"))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workloads", default=",".join(ALL))
    ap.add_argument("--extra", default="", help="extra bench.py flags, e.g. '--fc bf16 --no-cpu'")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    rows = []
    for w in args.workloads.split(","):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--steps",
               str(args.steps), "--warmup", str(args.warmup)] + args.extra.split()
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not line:
            rows.append({"workload": w, "error": (r.stderr or r.stdout)[-400:]})
            print(json.dumps(rows[-1]), flush=True)
            continue
        d = json.loads(line[-1])
        with open(os.path.join(args.out, f"sweep_{w}.json"), "w") as f:
            f.write(line[-1] + "\n")
        cb = d.get("cpu_baseline") or {}
        rows.append({
            "workload": w, "model": d["config"]["model"], "sla_s": d["config"]["sla_s"],
            "qps_at_sla": round(d["value"]), "mean_service_us": round(
                d["sla"]["mean_service_ms"] * 1e3, 1),
            "e2e_qps": round(d["e2e"]["value"]), "h2d_gbs": round(d["e2e"]["h2d_gbs"], 1),
            "roofline_bound": d["roofline"]["bound"], "roofline_kernel": d["roofline"]["kernel"],
            "roofline_achieved": round(d["roofline"]["achieved"], 1),
            "roofline_unit": d["roofline"]["unit"], "roofline_frac": round(d["roofline"]["frac"], 3),
            "cpu_deeprecsched_qps": round(cb.get("value", 0), 1), "cpu_cores": cb.get("cores"),
            "e2e_over_cpu": round(d["e2e"]["value"] / cb["value"], 1) if cb.get("value") else None,
            "clocks_sm_mhz": d["clocks"].get("sm_mhz")})
        print(json.dumps(rows[-1]), flush=True)
    with open(os.path.join(args.out, "summary.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
