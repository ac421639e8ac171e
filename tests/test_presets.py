"""The compiled launch-plan preset table against the autotune
record it was generated from, and its lookup through the C ABI."""
import json
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "paper_2405_15013_b200", "csrc", "ks_presets.inc")
# the table is generated from these records; later ones replace earlier rows with the same key
JSNS = [os.path.join(ROOT, "profiles", "r02", n) for n in ("autotune.json", "autotune_tf32_bsl.json", "autotune_fp32_bsf.json")]
JSNS.append(os.path.join(ROOT, "profiles", "r03", "autotune_tf32_bsf.json"))   # TF32 BSF re-tune after the TMA-store epilogue
JSNS.append(os.path.join(ROOT, "profiles", "r03", "autotune_tf32_bsf_v2.json"))  # ... and after MNJ / the d = 1 TMA store


def _rows():
    rows = {}
    for path in JSNS:
        for r in json.load(open(path))["rows"]:
            rows[(tuple(r["pattern"]), r["layout"], r["math"], r["lgB"])] = r
    return list(rows.values())


def _entries():
    pat = re.compile(r"^\{(\d+), (\d+), (\d+), (\d+), ([01]), ([01]), (\d+), (\d+)u\},")
    out = {}
    for line in open(INC):
        m = pat.match(line)
        if m:
            v = [int(x) for x in m.groups()]
            out[tuple(v[:7])] = v[7]
    return out


def test_table_matches_autotune_record():
    ent = _entries()
    rows = _rows()
    assert len(ent) >= 300
    for r in rows:
        a, b, c, d = r["pattern"]
        key = (a, b, c, d, 0 if r["layout"] == "bsf" else 1, 0 if r["math"] == "fp32" else 1, r["lgB"])
        assert ent[key] == r["best"]
        # a non-rule entry must have measured faster than the rules by the margin
        if r["best"] != r["rules"]:
            assert r["us"][str(r["best"])] < r["us"][str(r["rules"])]


def test_library_exports_table():
    import paper_2405_15013_b200 as ksb
    ksb.load_library()
    assert ksb.ks.preset_count() == len(_entries())


@pytest.mark.gpu
def test_preset_lookup_and_override():
    import numpy as np
    import torch
    import ksgen
    import paper_2405_15013_b200 as ksb
    from paper_2405_15013_b200 import ks
    B = ksgen.configs.SWEEP_BATCH
    p = (1, 48, 48, 2)
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1))
    k, src = f.plan_knobs(B, "bsf")
    assert src == 1 and k == _entries()[(1, 48, 48, 2, 0, 0, 14)]
    k2, src2 = f.plan_knobs(B + 100000, "bsf")          # another batch bucket: rules
    assert src2 == 0
    X = torch.from_numpy(ksgen.x_normal(B, p[0] * p[2] * p[3], seed=2)).cuda()
    Y1 = ksb.matmul(f, X)
    f.set_knobs(k2)                                        # the rules' knobs, forced
    assert f.plan_knobs(B, "bsf") == (k2, 2)
    Y2 = ksb.matmul(f, X)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)                             # FP32 knobs: bit-identical (R11)
    f.set_knobs(-1)
    with pytest.raises(ks.KSError):
        f.set_knobs(1 << 12)
