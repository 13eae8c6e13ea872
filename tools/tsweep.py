"""DeepRecSched on a B200: the UNMODIFIED reference scheduler (simulate /
max_qps_under_sla / tune, compiled from the reference sources into
oracle/_ref/librecsim_ref_b200.so) with accelerator service
times MEASURED on the GPU (rs_service_time through the link-time adapter),
against the same scheduler with the reference's modeled accelerator and
CPU-only. Sweeps the offload threshold T (the knob DeepRecSched tunes,
SURVEY §8d "T-sweep") and runs tune().

  python tools/tsweep.py [--models DLRM-RMC1,DLRM-RMC2,...] [--n 5000]

Test infrastructure on the reference side (oracle/ is test-only); the B200
side is the product library.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="DLRM-RMC1,DLRM-RMC2,DLRM-RMC3,WND,MT-WND,DIN,NCF")
    ap.add_argument("--n", type=int, default=5000)
    ap.add_argument("--thresholds", default="0,64,128,256,512,1000")
    ap.add_argument("--cpu", default="skylake")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_2001_02772_b200 as rs
    import oracle as orc
    dist = rs.SizeDistribution.production_heavy_tail()
    dist.max_size = 1000
    res = {"cpu_platform": args.cpu, "size_distribution": "production_heavy_tail (reference default)",
           "n": args.n, "batch": 64, "models": []}
    for name in args.models.split(","):
        spec = rs.builtin_model(name)
        if orc.load_ref_b200() is None:
            print(json.dumps({"error": "oracle/_ref/librecsim_ref_b200.so not built"}))
            return
        sla = rs.sla_target(name, "medium")
        row = {"model": name, "sla_s": sla, "sweep": []}
        for T in [int(x) for x in args.thresholds.split(",")]:
            cpu_only = T == 0
            b200 = orc.ref_max_qps(orc.load_ref_b200(), spec, "b200", args.cpu, sla, dist, args.n, 64,
                                   0 if cpu_only else T)
            modeled = orc.ref_max_qps(orc.load_ref_b200(), spec, "default", args.cpu, sla, dist, args.n,
                                      64, 0 if cpu_only else T)
            row["sweep"].append({"threshold": T, "qps_b200": b200[0], "p95_b200": b200[1],
                                 "accel_work_fraction_b200": b200[2], "qps_modeled_gpu": modeled[0],
                                 "accel_work_fraction_modeled": modeled[2]})
        row["tune_cpu_only"] = orc.ref_tune(orc.load_ref_b200(), spec, "", args.cpu, sla, dist, args.n)
        row["tune_modeled_gpu"] = orc.ref_tune(orc.load_ref_b200(), spec, "default", args.cpu, sla, dist,
                                               args.n)
        row["tune_b200"] = orc.ref_tune(orc.load_ref_b200(), spec, "b200", args.cpu, sla, dist, args.n)
        res["models"].append(row)
        print(json.dumps({"model": name, "tune_cpu_only_qps": row["tune_cpu_only"]["qps"],
                          "tune_modeled_gpu_qps": row["tune_modeled_gpu"]["qps"],
                          "tune_b200_qps": row["tune_b200"]["qps"],
                          "b200_threshold": row["tune_b200"]["threshold"]}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
