"""GPU run/verify harness: reference config format, variant names,
doc-id generator and CSV schema on the CPU; the verify grid and a bf16 run on the GPU."""
import numpy as np
import pytest

import pyoracle as O
from paper_2412_05496_b200 import harness as H


def test_config_text_and_json():
    cfg = H.parse_config_text("""
        # comment
        variant = causal, na_tiled(5,4), soft_cap(20)
        q_len = 256, 1024
        block_size = 64
        mode = forward, backward
        q_heads = 4
        kv_heads = 2
        seed = 0x10
    """, False)
    assert cfg.variants == ["causal", "na_tiled(5,4)", "soft_cap(20)"]
    assert cfg.q_lens == [256, 1024] and cfg.block_sizes == [64] and cfg.seed == 16
    cfg2 = H.parse_config_text('{"variant": ["alibi"], "q_len": [128], "mode": ["decode"]}', True)
    assert cfg2.variants == ["alibi"] and cfg2.modes == ["decode"]
    with pytest.raises(H.ConfigParse):
        H.parse_config_text("variant = causal\nq_len = 64\nmode = sideways", False)
    with pytest.raises(H.ConfigParse):
        H.parse_config_text("bogus_key = 1", False)


def test_variant_errors():
    with pytest.raises(H.UnknownVariant):
        H.make_variant("nonsense", 4, 256, 256, 1)
    with pytest.raises(H.ConfigParse):
        H.make_variant("sliding_window", 4, 256, 256, 1)       # missing argument
    with pytest.raises(H.ConfigParse):
        H.make_variant("na_naive(5)", 4, 250, 250, 1)          # not a square canvas
    with pytest.raises(H.ConfigParse):
        H.make_variant("sliding_window(2.5)", 4, 256, 256, 1)  # non-integer


@pytest.mark.parametrize("length,ndocs,seed", [(1000, 4, 0x5EED ^ 0xD0C5), (16384, 8, 0x5EED0001 ^ 0xD0C5)])
def test_doc_ids_match_reference_generator(length, ndocs, seed):
    assert np.array_equal(H.make_doc_ids(length, ndocs, seed), O.make_doc_ids(length, ndocs, seed))


def test_csv_schema():
    rows = [H.BenchRow("na_tiled(5,4)", 1, 4, 2, 256, 256, 64, 64, "forward", 123, 456, 0.25, 1e-7, 2e-8)]
    text = H.to_csv(rows, with_timing=False)
    lines = text.splitlines()
    assert lines[0] == H.CSV_HEADER
    assert lines[1] == '"na_tiled(5,4)",1,4,2,256,256,64,64,forward,0,456,0.25,1e-07,2e-08'


@pytest.mark.gpu
def test_gpu_verify_grid():
    rows = [r for g in H.VERIFY_GRIDS for r in H.run_bench(g, with_timing=False)]
    bad = [(r.variant, r.mode, r.block_size, r.detail) for r in rows if not r.ok]
    assert not bad, bad
    assert len(rows) == 10 * 3 * 2 + 10 * 4


@pytest.mark.gpu
def test_gpu_bf16_run_and_cli(tmp_path):
    out = tmp_path / "r.csv"
    rc = H.main(["run", "--variant", "sliding_window(300), alibi", "--qlen", "1024", "--mode", "forward",
                 "backward", "--dim", "128", "--dtype", "bf16", "--out", str(out)])
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0] == H.CSV_HEADER and len(lines) == 5
    assert H.main(["run", "--variant", "nonsense"]) == 1
