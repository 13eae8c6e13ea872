"""DeepRecSched's offload-threshold sweep at BASELINE configs[2] (DLRM-RMC2 /
RMC3, 32 tables x 10M rows x D=64), BOTH sides measured on this box
(VERDICT r1 item 7):

  * CPU requests: this host's cores, the oracle fp32 forward timed on requests
    of b items with 1 and all cores busy over 82 GB of materialised tables
    (oracle/cpu_arm.py) -> the reference's cpu_service_time is replaced by
    that table (oracle/ref_cpu_adapter.cpp);
  * offloaded queries: the B200 through the C-ABI (rs_service_breakdown via
    oracle/ref_b200_adapter.cpp: host-staged query, H2D + forward + D2H);
  * the scheduler: the UNMODIFIED reference (oracle/_ref/librecsim_ref_full.so)
    — max_qps_under_sla at the CPU-tuned batch B for every threshold T of
    tune()'s pow2 ladder (autotune.cpp:159-212), then tune() itself.

The reference has ONE accelerator FIFO (sim.cpp:95-97, 126-136): this sweep is
the K=1 system. K > 1 replicas are measured in real time by
`bench.py --serve --gpus K` (rs_serve), not simulated here.

  RS_B200_ROWS=10000000 python tools/cfg3_sweep.py > profiles/r2_cfg3_threshold_sweep.json
"""
import ctypes as C
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
P = C.POINTER


def main():
    os.environ.setdefault("RS_B200_ROWS", "10000000")
    import bench
    from oracle import OrModel, cpu_arm
    full = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "librecsim_ref_full.so"))
    full.ref_sweep_threshold.argtypes = [
        P(OrModel), C.c_char_p, C.c_char_p, C.c_double, C.c_uint64, C.c_int, C.c_double,
        C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64, P(C.c_int64),
        C.c_int64, P(C.c_double), P(C.c_double), P(C.c_double)]
    full.ref_tune.argtypes = cpu_arm.ref_cpu.ref_tune.argtypes
    mu, sigma = math.log(300), 0.5
    ladder = [0, 1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1000]
    out = {"size_distribution": "LogNormal(ln 300, 0.5) clamped [1, 1000]", "n": 50_000,
           "cpu": "this host, measured (all cores)", "accelerator": "1 x B200, measured",
           "workloads": []}
    for wl in ("cfg3-rmc2", "cfg3-rmc3"):
        m, rows, zoo = bench.workload_or_model(wl)
        sla = cpu_arm.sla_target(zoo)
        t0 = time.time()
        arm = cpu_arm.CpuDeepRecSched(m, rows)
        for _ in range(3):
            arm.sample(4.0)
        cpu_only = arm.tune(sla, mu, sigma)
        arm.install(full)
        B = cpu_only["batch"]
        T = (C.c_int64 * len(ladder))(*ladder)
        q = (C.c_double * len(ladder))()
        p = (C.c_double * len(ladder))()
        f = (C.c_double * len(ladder))()
        rc = full.ref_sweep_threshold(C.byref(m), b"measured", b"b200", sla, 42,
                                      cpu_arm.LOGNORMAL, mu, sigma, 0.0, 0.0, 1000, 50_000, B,
                                      T, len(ladder), q, p, f)
        if rc:
            raise RuntimeError(f"ref_sweep_threshold rc={rc}")
        b, t, steps = C.c_int64(), C.c_int64(), C.c_int64()
        tq, tp, tf = C.c_double(), C.c_double(), C.c_double()
        rc = full.ref_tune(C.byref(m), b"measured", b"b200", sla, 42, cpu_arm.LOGNORMAL, mu,
                           sigma, 0.0, 0.0, 1000, 50_000, 1, C.byref(b), C.byref(t),
                           C.byref(tq), C.byref(tp), C.byref(tf), C.byref(steps))
        if rc:
            raise RuntimeError(f"ref_tune rc={rc}")
        bs, t1, tc = arm.table()
        arm.close()
        rec = {"workload": wl, "rows_per_table": rows, "sla_s": sla,
               "cpu_request_table": {"items": bs.tolist(), "s_1core": t1.tolist(),
                                     "s_all_cores": tc.tolist(), "cores": arm.threads},
               "cpu_only_tune": cpu_only,
               "sweep_at_batch": B,
               "sweep": [{"threshold": ladder[i], "qps": q[i], "p95_ms": p[i] * 1e3,
                          "accel_work_fraction": f[i]} for i in range(len(ladder))],
               "tune_cpu_plus_b200": {"batch": b.value, "threshold": t.value, "qps": tq.value,
                                      "p95_ms": tp.value * 1e3, "accel_work_fraction": tf.value,
                                      "search_steps": steps.value},
               "wall_s": time.time() - t0}
        out["workloads"].append(rec)
        print(wl, json.dumps({"cpu_only": cpu_only["qps"], "tuned": rec["tune_cpu_plus_b200"]}),
              file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
