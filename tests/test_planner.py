"""Block-size planner (include/distr_attn.h distr_attn_plan): the B200 analogue of §3.3.1
(P:320-369). Host-only — runs without a GPU."""
import pytest

import paper_2507_17245_b200 as da
from paper_2507_17245_b200 import DistrAttnError
from paper_2507_17245_b200.build import build

build()

ENVELOPE = [(d, l, g) for d in (32, 64, 128) for l in (64, 128) for g in (1, 2, 4, 8)
            if d % g == 0 and d // g >= 16 and (128 // l) * d // g <= 128]


@pytest.mark.parametrize("d,l,g", ENVELOPE)
def test_plan_respects_b200_budgets(d, l, g):
    p = da.distr_attn_plan(16384, d, block_l=l, group_size=g)
    # Eq. 4 analogue: tiles are whole tcgen05 shapes (M = 128; N multiple of 16, <= 256)
    assert p["tile_m"] == 128 and p["tile_n"] % 16 == 0 and p["tile_n"] <= 256
    # the contraction width of S is the reduced one: (128 / l) * d / G* (block-diagonal for l=64)
    assert p["s_width"] == (128 // l) * d // g
    # Eq. 5 analogue: two Q tiles in flight, within TMEM (512 columns) and smem (227 KB)
    assert p["tiles_per_cta"] == 2
    assert p["tiles_per_cta"] * (d + p["tile_n"]) <= p["tmem_cols"] == 512
    assert p["tile_n"] <= p["m_max_tmem"]
    assert p["smem_bytes"] <= 232448
    assert p["kv_stages"] >= 1 and p["khat_stages"] >= 1
    assert p["threads"] == 512


def test_exact_plan():
    p = da.distr_attn_plan(16384, 128, distr=False)
    assert p["s_width"] == 128 and p["khat_stages"] == 0 and p["threads"] == 384
    assert p["fusion_smem_bytes_per_tile"] == 0


def test_per_tile_budgets_match_survey_table():
    # SURVEY §8(d) per-tile budget (clk per SM): exact d=128 MMA 1024, G*=2 768, G*=4 640;
    # d=64 exact 512, G*=2 384; MUFU 1024 for every 128 x 128 tile
    assert da.distr_attn_plan(4096, 128, distr=False)["mma_clk_per_tile"] == 1024
    assert da.distr_attn_plan(4096, 128, group_size=2)["mma_clk_per_tile"] == 768
    assert da.distr_attn_plan(4096, 128, group_size=4)["mma_clk_per_tile"] == 640
    assert da.distr_attn_plan(4096, 64, distr=False)["mma_clk_per_tile"] == 512
    assert da.distr_attn_plan(4096, 64, group_size=2)["mma_clk_per_tile"] == 384
    assert da.distr_attn_plan(4096, 64, group_size=2)["exp_clk_per_tile"] == 1024


def test_paper_io_model():
    # I(l, m) = N/l (ld + 2Nd + ld) — larger l always means less I/O, m does not enter
    N, d = 8192, 64
    i64 = da.distr_attn_plan(N, d, block_l=64)["hbm_bytes_paper"]
    i128 = da.distr_attn_plan(N, d, block_l=128)["hbm_bytes_paper"]
    assert i128 < i64
    assert i128 == 2 * (N / 128) * (128 * d + 2 * N * d + 128 * d)
    # on B200 the K/V re-reads hit L2: HBM ~ Q, K, V, O once (+ K^T pass for distr)
    assert da.distr_attn_plan(N, d, distr=False)["hbm_bytes_b200"] == 2 * 4 * N * d
    assert da.distr_attn_plan(N, d)["hbm_bytes_b200"] == 2 * 6 * N * d


def test_tmem_bound_on_m():
    # tiles * (d + m) <= 512: d=128 leaves m <= 128, d=64 leaves m <= 192
    assert da.distr_attn_plan(4096, 128)["m_max_tmem"] == 128
    assert da.distr_attn_plan(4096, 64)["m_max_tmem"] == 192
    assert da.distr_attn_plan(4096, 32)["m_max_tmem"] == 224


def test_ctas_cover_all_q_tiles():
    for N in (1, 255, 256, 257, 16384):
        assert da.distr_attn_plan(N, 128)["ctas"] == (N + 255) // 256


@pytest.mark.parametrize("args,status", [((0, 128, 128, 2), 1), ((4096, 96, 128, 2), 2),
                                         ((4096, 64, 128, 3), 2), ((4096, 64, 128, 8), 2),
                                         ((4096, 128, 32, 2), 2)])
def test_plan_rejects_unsupported(args, status):
    N, d, l, g = args
    with pytest.raises(DistrAttnError) as e:
        da.distr_attn_plan(N, d, block_l=l, group_size=g)
    assert e.value.status == status


@pytest.mark.parametrize("d,g", [(32, 2), (64, 2), (64, 4), (128, 2), (128, 4)])
def test_plan_block256_shares_one_grouping_per_cta(d, g):
    # block_l = 256 = the two Q tiles of one CTA: S width d/G* (no stacking), one fused K̂ per key
    # tile for both tiles (half the fusion traffic of block_l = 128), within the smem budget
    p = da.distr_attn_plan(16384, d, block_l=256, group_size=g)
    q = da.distr_attn_plan(16384, d, block_l=128, group_size=g)
    assert p["s_width"] == q["s_width"] == d // g
    assert p["fusion_smem_bytes_per_tile"] == q["fusion_smem_bytes_per_tile"] / 2
    assert p["smem_bytes"] <= 232448 and p["khat_stages"] >= 1
    # the paper's I/O model prefers the larger block
    assert p["hbm_bytes_paper"] < q["hbm_bytes_paper"]


# ------------------------------------------------------------------------------ distr_attn_choose
# The choosing planner against the measured sweeps committed under profiles/ (tools/sweep.py,
# block_l 128 and 256, G* 2 and 4, and the own exact kernel): for every BASELINE config and C4
# sweep point, the setting it picks must measure within 5 % of the fastest measured setting
# (5 % = the run-to-run spread of these timings on one box).
import glob
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILE = sorted(p for p in glob.glob(os.path.join(ROOT, "profiles", "r02_v*"))
                 if os.path.exists(os.path.join(p, "sweep.json")) and os.path.exists(os.path.join(p, "sweep_l256.json")))[-1]


def measured():
    rows = {}
    for name in ("sweep.json", "sweep_l256.json"):
        for line in open(os.path.join(PROFILE, name)):
            r = json.loads(line)
            key = (r["B"], r["H"], r["H_kv"], r["N"], r["d"], r["causal"], r["dtype"])
            rows.setdefault(key, {})[("exact", 0, 1)] = min(
                rows.get(key, {}).get(("exact", 0, 1), 1e9), r["exact_ms"])
            rows[key][("distr", r["block_l"], r["G"])] = r["distr_ms"]
    return rows


@pytest.mark.parametrize("key", sorted(measured()))
def test_choice_is_within_noise_of_the_fastest_measured(key):
    B, H, Hkv, N, d, causal, dtype = key
    cand = measured()[key]
    c = da.distr_attn_choose(B, H, Hkv, N, d, causal=causal, max_group_size=4)
    pick = ("distr", c["block_l"], c["group_size"]) if c["distr"] else ("exact", 0, 1)
    if pick not in cand:  # a setting the sweep did not run at this shape (e.g. block_l=64)
        pytest.skip(f"{pick} not measured at {key}")
    best = min(cand.values())
    assert cand[pick] <= 1.05 * best, (key, pick, cand)


def test_choice_respects_the_accuracy_bound_and_envelope():
    for N in (4096, 65536):
        for mg in (1, 2, 4, 8):
            c = da.distr_attn_choose(1, 16, 16, N, 128, max_group_size=mg)
            assert c["group_size"] <= max(1, mg)
            if mg == 1:
                assert c["distr"] == 0  # G* = 1 is exact attention: nothing to gain
            assert c["predicted_us"] == min(c["predicted_exact_us"], c["predicted_distr_us"])
    assert da.distr_attn_choose(1, 1, 1, 4096, 32, max_group_size=8)["group_size"] <= 2  # d/G* >= 16
    with pytest.raises(DistrAttnError):
        da.distr_attn_choose(1, 3, 2, 128, 128)
