"""Host-side bench accounting (no GPU): the per-direction byte split used by
the direction-aware HBM model adds up to the algorithmic bytes of SURVEY
8(d) for every BASELINE configuration and shard size."""
import bench
import synth


def test_rw_bytes_sum_to_algorithmic_bytes():
    for name, cfg in synth.CONFIGS.items():
        for R in (1, 7, cfg["R"]):
            alg = bench.algorithmic_bytes(cfg, R)
            rw = bench.rw_bytes(cfg, R)
            assert set(rw) == set(alg), name
            for k, (rd, wr) in rw.items():
                assert rd + wr == alg[k], (name, R, k)
                assert rd > 0 and wr > 0


def test_rw_bytes_directions():
    cfg = synth.CONFIGS["c4"]
    R, F, H = cfg["R"], cfg["F"], cfg["H"]
    rw = bench.rw_bytes(cfg, R)
    n = R * F
    assert rw["act_fwd"] == (2 * n, 2 * n + n // 4)        # read x; write y + codes
    assert rw["act_bwd"] == (2 * n + n // 4, 2 * n)        # read dy + codes; write dx
    assert rw["norm_fwd"] == (2 * R * H, 2 * R * H + 4 * R)
    assert rw["norm_bwd"] == (4 * R * H + 4 * R, 2 * R * H)
