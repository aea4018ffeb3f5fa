"""fetch_cost calibration: measured link specs are
sane and the reference's own cost model, fed with them, predicts the real
gather time of a mixed local/host batch within 25% (the tier-isolated
gather runs the local and host reads concurrently, which is the model's
max-over-locations tail rule)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_calibrated_links_predict_gather(qvb):
    import torch

    from paper_2305_10863_b200 import calibrate

    t = calibrate.calibrated_topology()
    loc_bw = t.link_bandwidth_Bps[qvb.LINK_LOCAL]
    pcie_bw = t.link_bandwidth_Bps[qvb.LINK_PCIE]
    assert 1e12 < loc_bw < 8e12, loc_bw  # HBM-scale
    assert 5e9 < pcie_bw < 70e9, pcie_bw  # PCIe Gen5 x16 scale
    assert 0 < t.link_latency_s[qvb.LINK_LOCAL] < 1e-3

    # 30% of rows on the host: the model's max-over-locations tail rule
    n, dim, b = 1 << 20, 128, 1 << 18
    t.gpus_per_server = 1
    t.gpu_feature_capacity = int(n * 0.7)
    t.host_feature_capacity = n
    lo, ids = qvb.plan_placement(np.random.default_rng(3).random(n), t)
    loc, off = qvb.build_lookup_table(lo, ids, t)
    store = qvb.FeatureStore(lo, ids, dim, t, reader=0)
    req = torch.empty(b, dtype=torch.int64, device="cuda")
    qvb.request_ids_synthetic(11, 5, n, req)
    out = torch.empty((b, dim), dtype=torch.float32, device="cuda")
    measured = calibrate._time_gather(store, req, out, reps=5)
    plan = qvb.plan_reads(loc, off, req.cpu().numpy().view(np.uint64), 8)
    t.tlb_miss_penalty_s = 0.0  # zero-copy reads are not page-walk bound here
    predicted = calibrate.fetch_cost(plan[:3], t, dim * 4)
    store.close()
    assert 0.75 * predicted < measured < 1.25 * predicted, (predicted, measured)
