"""The seeded input generator (R12): SplitMix64 reference outputs and
the ranges / shapes of the five BASELINE.json configurations."""
import numpy as np

import synth


def test_splitmix64_reference_values():
    # SplitMix64 with seed 0 (Steele et al. 2014; the widely published first outputs)
    g = synth.SplitMix64(0)
    assert [g.next() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_block_equals_sequential():
    a = synth.SplitMix64(42).next_block(100)
    g = synth.SplitMix64(42)
    assert [int(v) for v in a] == [g.next() for _ in range(100)]


def test_configs_ranges():
    for name, cfg in synth.CONFIGS.items():
        small = name in ("c256", "c512", "ml")
        I = synth.make_instance(cfg, m=min(cfg.m, 16), n=min(cfg.n, 16), l=min(cfg.l, 16)) if small \
            else synth.make_instance(cfg)
        lo, hi = cfg.a_range
        assert I.A.min() >= lo and I.A.max() <= hi and I.A.dtype == (np.int8 if cfg.signed else np.uint8)
        assert I.B.min() >= cfg.b_lo and I.B.max() <= cfg.b_hi
        assert 1 <= I.x < synth.P256_ORDER
        r = [int.from_bytes(v.tobytes(), "big") for v in I.r_be]
        assert all(1 <= v < synth.P256_ORDER for v in r)


def test_keygen_secret_is_first_draw():
    assert synth.keygen_secret(3) == synth.make_instance(synth.CONFIGS["c512"], m=2, n=2, l=2).x
