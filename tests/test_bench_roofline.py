"""bench.py's roofline denominators (-m "not gpu"): the primary peak of a derived-ratio dtype is the
highest rate measured for it (nominal ratio x MEASURED_PEAKS bf16, same-run library, power-capped
MMA-only probe), BF16 keeps MEASURED_PEAKS' own number, and every candidate is listed."""
import types

import bench

PK = {"bf16": 1605.0, "hbm": 6546.6, "source": "MEASURED_PEAKS.json", "bf16_sustained": 1300.0}


def _work(kind, flops, cfg="cX"):
    return types.SimpleNamespace(bound="tensor", kind=kind, flops=flops, cfg=cfg, kernel="k", sm_mhz_eff=1300.0)


def test_bf16_keeps_measured_peak():
    w = _work("bf16", 2.0 * 8192 ** 3)
    ms = w.flops / 1500e12 * 1e3                       # 1500 TFLOP/s
    rl = bench.roofline(w, ms, PK, {"reasons": []}, anchor=1650.0)
    assert rl["peak"] == 1605.0 and abs(rl["frac"] - 1500 / 1605) < 1e-3
    bench.apply_power_roofline(rl, 1745.0, "bf16")
    assert rl["peak"] == 1605.0                         # contract: MEASURED_PEAKS for bf16
    assert abs(rl["denominators"]["power_capped_mma_only"]["frac"] - 1500 / 1745) < 1e-3
    assert rl["denominators"]["same_run_library"]["peak"] == 1650.0


def test_derived_ratio_takes_highest_measured():
    w = _work("tf32", 2.0 * 8192 ** 3)
    ms = w.flops / 850e12 * 1e3                        # 850 TFLOP/s > 0.5 x 1605
    rl = bench.roofline(w, ms, PK, {"reasons": []}, anchor=762.0)
    assert rl["peak"] == 802.5 and rl["frac"] > 1.0    # the nominal ratio alone is beaten
    bench.apply_power_roofline(rl, 954.0, "tf32")
    assert rl["peak"] == 954.0 and rl["frac"] < 1.0 and "power-capped" in rl["peak_source"]
    # a library anchor above both wins the same way
    rl2 = bench.roofline(w, ms, PK, {"reasons": []}, anchor=1000.0)
    bench.apply_power_roofline(rl2, 954.0, "tf32")
    assert rl2["peak"] == 1000.0 and "library" in rl2["peak_source"]


def test_power_kinds_cover_tensor_configs():
    # every non-bf16 tensor kind the bench times has a probe configuration
    for kind in ("tf32", "s8", "sp16", "sp8", "sptf32"):
        assert kind in bench._POWER_KINDS and kind in bench.KIND_RATIO
