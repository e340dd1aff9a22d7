"""Parameter selection (paper_2002_03258_b200.tuning): plans for the BASELINE shapes and the
tuning knobs, host-side only (no GPU needed)."""

import pytest

from paper_2002_03258_b200 import tuning


def test_plan_config2_tsm2r():
    p = tuning.plan("double", 30720, 30720, 8)
    assert p["impl"] == "tma" and p["consumer"] == "dmmap"  # fp64 8-column passes, pipelined (envab_r01.json)
    assert p["t1"] == 512 and p["t2"] == 8 and p["t3"] == 48
    assert p["grid"] <= 148 and p["items"] >= 8 * p["grid"]  # ~10 items per CTA (8 MB big, 1 MB small)
    assert p["nbig"] > 0 and p["nsmall"] > 0 and p["batch"] == 1
    # the small items cover roughly the last 10% of each row block's columns (DMMA passes)
    assert 0.08 <= p["nsmall"] * p["ksmall"] / 30720 <= 0.2
    # fp64 3-4 column passes run on the DMMA kernel's 8-column tile (swizzle_r01.txt); n=2 stays on
    # DFMA and keeps the 20 % tail
    p4 = tuning.plan("double", 30720, 30720, 4)
    assert p4["consumer"] == "dmmap" and p4["cols_per_pass"] == 8
    assert tuning.plan("double", 30720, 30720, 2)["nsmall"] * tuning.plan("double", 30720, 30720, 2)["ksmall"] \
        >= 0.15 * 30720
    tuning.set_tuning(tuning.Tuning(consumer=1))
    try:
        assert tuning.plan("double", 30720, 30720, 4)["consumer"] == "fma"  # a forced consumer keeps the 4-column pass
    finally:
        tuning.set_tuning(None)


@pytest.mark.parametrize("mk,n,prec", [(2048, 16, "double"), (4096, 8, "double"), (6144, 16, "double"),
                                       (8192, 8, "double"), (4096, 16, "single")])
def test_plan_midsize_one_item_per_cta(mk, n, prec):
    # mid-size problems: equal column ranges, no small-item tail; up to ~4 MB of A per CTA that is
    # one round of at most one item per CTA (ncu cold and sustained A/B: profiles/midsize_r01.jsonl)
    p = tuning.plan(prec, mk, mk, n)
    assert p["items"] == p["grid"] <= 148 and p["items"] >= 100
    assert p["nbig"] == 0 and p["kbig"] == p["ksmall"] and p["ksmall"] % p["cols_per_stage"] == 0
    rb = -(-mk // p["rows_per_block"])
    assert rb * -(-mk // p["ksmall"]) == p["items"]
    # the knobs still override it, and large problems keep the big-item + tail split
    tuning.set_tuning(tuning.Tuning(small_kb=256))
    try:
        assert tuning.plan(prec, mk, mk, n)["items"] != p["items"] or mk == 2048
    finally:
        tuning.set_tuning(None)
    assert tuning.plan(prec, 30720, 30720, n)["nbig"] > 0


def test_plan_few_row_blocks_split():
    # fewer row blocks than CTAs: short-k shapes are split across CTAs too (fp32 512^2 x 16 used
    # to run on one CTA), while TSM2L shapes (k within one stage) stay single-chunk
    p = tuning.plan("single", 512, 512, 16)  # small C += call: FFMA2, fp32 reductions into C
    assert p["consumer"] == "ffma2" and p["items"] == p["grid"] == p["nsmall"] > 16
    p = tuning.plan("double", 1000, 200, 8)
    assert p["nsmall"] > 1 and p["grid"] == p["items"]
    p = tuning.plan("double", 4096, 16, 16)
    assert p["nsmall"] == 1 and p["items"] == 8
    assert tuning.plan("double", 51200, 64, 8)["nsmall"] == 1  # 100 row blocks: splitting buys nothing


def test_plan_midsize_rounds():
    # larger mid-size problems: a few equal rounds (16384^2: 32 row blocks x 9 pieces on 148 CTAs)
    p = tuning.plan("double", 16384, 16384, 8)
    assert p["nbig"] == 0 and p["items"] == 288 and p["grid"] == 148
    assert p["nsmall"] * p["ksmall"] >= 16384 > (p["nsmall"] - 1) * p["ksmall"]


def test_plan_tsm2l_single_chunk():
    p = tuning.plan("double", 1 << 24, 16, 16)
    assert p["impl"] == "tma" and p["consumer"] == "dmma"  # fp64 16-column passes (abtest_r01e.json)
    assert p["nbig"] == 0 and p["nsmall"] == 1 and p["batch"] == 1  # 64 KB grabs = one 512x16 row block
    assert tuning.plan("double", 1 << 24, 4, 16)["batch"] == 4
    assert tuning.plan("double", 1 << 24, 16, 8)["consumer"] == "dmma"
    assert tuning.plan("double", 1 << 24, 16, 4)["consumer"] == "dmma"  # 8-column DMMA tile
    assert tuning.plan("double", 1 << 24, 16, 2)["consumer"] == "fma"


def test_plan_fp32_and_wide():
    p = tuning.plan("single", 32768, 32768, 16)
    assert p["consumer"] == "tc" and p["t1"] == 512 and p["cols_per_stage"] == 16  # tcgen05 split tf32
    assert tuning.plan("single", 32768, 32768, 8)["consumer"] == "ffma2"
    # TSM2L shapes (single-chunk row blocks): FFMA2 with direct stores, not the tensor cores
    assert tuning.plan("single", 1 << 24, 16, 16)["consumer"] == "ffma2"
    assert tuning.plan("single", 1 << 24, 16, 16)["nbig"] + tuning.plan("single", 1 << 24, 16, 16)["nsmall"] == 1
    p = tuning.plan("single", 32768, 32768, 16, deterministic=True)  # ordered combine stays on FFMA2
    assert p["consumer"] == "ffma2" and p["t1"] == 1024
    assert tuning.plan("single", 1001, 5000, 16, lda=1004)["consumer"] == "ffma2"  # lda < roundup(m, 32)
    assert tuning.plan("double", 1000, 1000, 40)["passes"] == 3


def test_plan_fallbacks():
    assert tuning.plan("double", 1001, 5000, 8, lda=1001)["impl"] == "ldg"     # odd lda: no TMA
    assert tuning.plan("double", 1001, 16, 8, lda=1001)["impl"] == "tsm2l"
    assert tuning.plan("double", 4096, 4096, 8, deterministic=True)["deterministic"] == 1
    assert tuning.plan("double", 4096, 4096, 8, impl="ablation")["impl"] == "ablation"


def test_tuning_knobs_round_trip_and_change_the_plan():
    base = tuning.plan("double", 30720, 30720, 8)
    try:
        tuning.set_tuning(tuning.Tuning(consumer=1, small_kb=128, big_kb=2048, tail_pct=40))
        assert tuning.get_tuning() == tuning.Tuning(consumer=1, small_kb=128, big_kb=2048, tail_pct=40)
        p = tuning.plan("double", 30720, 30720, 8)
        assert p["consumer"] == "fma"
        assert p["ksmall"] == 128 * 1024 // (512 * 8)
        assert p["kbig"] == 2048 * 1024 // (512 * 8)
        assert p["nsmall"] * p["ksmall"] >= 0.4 * 30720 - p["ksmall"]
        assert p["items"] != base["items"]
        with pytest.raises(ValueError):
            tuning.set_tuning(tuning.Tuning(tail_pct=101))
    finally:
        tuning.set_tuning(None)
    assert tuning.get_tuning() == tuning.Tuning()
    assert tuning.plan("double", 30720, 30720, 8) == base


def test_all_consumer_knobs_accepted():
    for c in range(6):
        try:
            tuning.set_tuning(tuning.Tuning(consumer=c))
            assert tuning.get_tuning().consumer == c
        finally:
            tuning.set_tuning(None)
    with pytest.raises(ValueError):
        tuning.set_tuning(tuning.Tuning(consumer=6))
    tuning.set_tuning(None)
