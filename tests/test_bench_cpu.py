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


class _FakeWorkload:
    """Outputs of rows [row0, row0 + R) of a global (all-rows) output set."""

    def __init__(self, cfg, full, row0, R):
        import torch
        self.cfg = cfg
        sl = bench.row_slices(cfg, row0, row0 + R)
        for name in bench.OUTPUTS:
            lo, hi = sl[name]
            setattr(self, name, full[name].reshape(-1)[lo:hi].clone())


def _full_outputs(cfg, R, seed=0):
    import torch
    g = torch.Generator().manual_seed(seed)
    F, H = cfg["F"], cfg["H"]
    return {"y": torch.randn(R, F, generator=g).to(torch.bfloat16),
            "codes": torch.randint(0, 256, (R * F // 4,), generator=g, dtype=torch.uint8),
            "dx": torch.randn(R, F, generator=g).to(torch.bfloat16),
            "yn": torch.randn(R, H, generator=g).to(torch.bfloat16),
            "rstd": torch.rand(R, generator=g),
            "dxn": torch.randn(R, H, generator=g).to(torch.bfloat16)}


def test_shard_checksums_match_one_gpu_and_catch_a_flipped_or_moved_byte():
    """8(e) shard invariance in the bench: each rank's checksums of its row
    block equal rank 0's checksums of the same rows of the one-GPU run; a
    single flipped bit, or two swapped bytes, in any output changes them."""
    cfg = dict(synth.CONFIGS["c5"], F=64, H=32)
    R, world = 24, 4
    full = _full_outputs(cfg, R)
    one = _FakeWorkload(cfg, full, 0, R)
    for rank in range(world):
        r0, n = bench.shard_rows(R, world, rank, "strong")
        shard = _FakeWorkload(cfg, full, r0, n)
        assert bench.output_checksums(shard, r0, r0 + n, r0) == bench.output_checksums(one, r0, r0 + n, 0)
    r0, n = bench.shard_rows(R, world, 2, "strong")
    ref = bench.output_checksums(_FakeWorkload(cfg, full, r0, n), r0, r0 + n, r0)
    for i, name in enumerate(bench.OUTPUTS):
        for mutate in ("flip", "swap"):
            bad = {k: v.clone() for k, v in full.items()}
            raw = bad[name].reshape(-1).view(__import__("torch").uint8)
            lo, hi = bench.row_slices(cfg, r0, r0 + n)[name]
            eb = bad[name].element_size()
            j = lo * eb + 3
            if mutate == "flip":
                raw[j] ^= 1
            else:
                if raw[j] == raw[j + 1]:
                    raw[j + 1] ^= 0x80
                raw[j], raw[j + 1] = raw[j + 1].clone(), raw[j].clone()
            got = bench.output_checksums(_FakeWorkload(cfg, bad, r0, n), r0, r0 + n, r0)
            assert got[i] != ref[i], (name, mutate)


def test_stream_sets_keep_every_buffer_cold():
    """The in-stream protocols' set count: a kernel launched back to back with
    itself over N sets touches a buffer again only after (N - 1) launches,
    which must be >= 3 x L2 bytes for the smallest kernel of every config."""
    l2 = 126 << 20
    for name, cfg in synth.CONFIGS.items():
        nb = bench.algorithmic_bytes(cfg, cfg["R"])
        n = bench.stream_sets(nb, l2)
        assert n >= 2
        if n < 256:
            assert (n - 1) * min(nb.values()) >= 3 * l2, name
