"""The drop-in claim, end to end: the UNMODIFIED reference scheduler
(simulate / max_qps_under_sla / tune, compiled from /root/reference sources
into oracle/_ref) runs against the B200 path through the link-time adapter
oracle/ref_b200_adapter.cpp. With AcceleratorSpec "b200" the
reference's accel_service_time is answered by rs_service_time (measured on the
GPU); every other spec keeps the reference's modeled cost."""
import math

import pytest

import paper_2001_02772_b200 as rs


def _libs(orc):
    if orc.ref is None or orc.load_ref_b200() is None:
        pytest.skip("oracle/_ref libraries not built (no /root/reference here)")
    return orc.ref, orc.load_ref_b200()


def test_wrapped_library_keeps_reference_behaviour_for_other_specs(orc):
    ref, ref_b200 = _libs(orc)
    spec = rs.builtin_model("DLRM-RMC1")
    dist = rs.SizeDistribution.production_heavy_tail()
    a = orc.ref_max_qps(ref, spec, "default", "skylake", 0.1, dist, 2000, 64, 324)
    b = orc.ref_max_qps(ref_b200, spec, "default", "skylake", 0.1, dist, 2000, 64, 324)
    assert a == b


@pytest.mark.gpu
def test_reference_simulate_runs_on_measured_b200_service_times(orc):
    _, ref_b200 = _libs(orc)
    spec = rs.builtin_model("DLRM-RMC1")
    dist = rs.SizeDistribution.production_heavy_tail()
    cpu_only = orc.ref_max_qps(ref_b200, spec, "default", "skylake", 0.1, dist, 3000, 64, 0)
    modeled = orc.ref_max_qps(ref_b200, spec, "default", "skylake", 0.1, dist, 3000, 64, 324)
    b200 = orc.ref_max_qps(ref_b200, spec, "b200", "skylake", 0.1, dist, 3000, 64, 324)
    assert b200[0] > cpu_only[0]            # offloading to the B200 raises QPS
    assert b200[0] >= modeled[0]            # and beats the modeled 1080Ti-class device
    assert 0 < b200[2] < 1                  # some, not all, work offloaded at T=324


@pytest.mark.gpu
def test_deeprecsched_tunes_b200_thresholds(orc):
    """Phase 2 of tune() (autotune.cpp:159-212) climbs the offload threshold
    with measured B200 service times and adopts the accelerator."""
    _, ref_b200 = _libs(orc)
    spec = rs.builtin_model("DLRM-RMC1")
    dist = rs.SizeDistribution.production_heavy_tail()
    dist.max_size = 1000
    cpu = orc.ref_tune(ref_b200, spec, "", "skylake", 0.1, dist, 1500)
    b200 = orc.ref_tune(ref_b200, spec, "b200", "skylake", 0.1, dist, 1500)
    assert cpu["threshold"] == 0
    assert b200["threshold"] > 0 and b200["qps"] >= cpu["qps"]
    assert math.isfinite(b200["p95"]) and b200["p95"] <= 0.1


@pytest.mark.gpu
def test_adapter_returns_whole_service_time_and_reference_exceptions(orc):
    """The adapter answers the reference's accel_service_time with the whole
    measured ServiceTime (total, transfer, per-category compute summing to
    total - transfer) and maps RS_E_* failures to the reference's exception
    types: a query above the handle's 1000-item capacity (RS_E_CAPACITY) is a
    std::invalid_argument (shim code -1), as S < 1 is in the reference
    (platform.cpp:115). Two inline specs with the same name but different
    shapes get different handles (keyed by shape)."""
    _, ref_b200 = _libs(orc)
    spec = rs.builtin_model("DLRM-RMC3")
    rc, total, transfer, pc = orc.ref_accel_service_time(ref_b200, spec, "b200", 200)
    assert rc == 0 and 0 < transfer < total < 0.1
    assert abs(sum(pc) - (total - transfer)) <= 1e-9 + 1e-6 * total
    assert orc.ref_accel_service_time(ref_b200, spec, "b200", 1001)[0] == -1
    assert orc.ref_accel_service_time(ref_b200, spec, "b200", 0)[0] == -1
    # the modeled accelerator still takes the reference's own path
    rc, total_d, transfer_d, _ = orc.ref_accel_service_time(ref_b200, spec, "default", 200)
    assert rc == 0 and transfer_d > 0
    other = rs.ModelSpec("DLRM-RMC3", dense_fc=rs.LayerStack([64, 32]),
                         predict_fc=rs.LayerStack([64, 1]),
                         embeddings=rs.EmbeddingConfig(4, 5, 32, "Sum"), dense_input_dim=16)
    rc2, total2, _, _ = orc.ref_accel_service_time(ref_b200, other, "b200", 200)
    assert rc2 == 0 and total2 != total  # a different shape, its own handle
