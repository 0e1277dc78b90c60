"""Host-side roofline bookkeeping (not gpu): the paper's RTX-4090 crossovers and B200 figures."""
from paper_2505_05799_b200.roofline import block_roofline, crossover_m, layer_roofline, load_peaks


def test_4090_crossovers_match_paper():
    # public RTX 4090 peaks: fp16 w/ fp32 accumulate 165.2 TFLOP/s, 1008 GB/s
    p, bw = 165.2e12, 1008e9
    assert round(crossover_m(p, 1.0, bw)) == 82    # W4A16 vs W8A8: paper says A < 83
    assert round(crossover_m(p, 0.5, bw)) == 41    # W2A16 vs W4A4: paper says A < 42


def test_b200_crossovers():
    pk = load_peaks()
    m = crossover_m(pk["bf16_tflops"] * 1e12, 1.0, pk["hbm_gbs"] * 1e9)
    assert 100 < m < 150  # 124 with the measured peaks


def test_block_roofline_bounds():
    pk = {"bf16_tflops": 1000.0, "i8_tops": 2000.0, "hbm_gbs": 1000.0}
    r = block_roofline(1, 4096, 4096, 4, 16, 128, False, pk)
    assert r["t"] == r["bytes"] / 1e12  # m = 1: memory-bound
    r = block_roofline(8192, 4096, 4096, 8, 8, -1, True, pk)
    assert r["t"] == r["flops"] / 2e15  # large m: int8 compute-bound
