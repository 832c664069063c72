"""CPU checks of the boundary: the C-ABI library loads, exports every symbol the header
declares, validates arguments before touching the GPU, and the sharding host logic."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "bkfac.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bkfac_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2210_08494_b200 import binding
    return binding.load()


def test_exports_every_declared_symbol(lib):
    names = _header_functions()
    assert "bkfac_brand_update" in names and "bkfac_precondition" in names
    for name in names:
        assert hasattr(lib, name), f"missing export {name}"
    from paper_2210_08494_b200 import binding
    assert sorted(binding.EXPORTED) == names


def test_binding_constants_match_header():
    """Every #define of include/bkfac.h that the binding mirrors (options, GEMM paths, factor
    flags) has the same value on both sides, and every BKFAC_OPT_* of the header is mirrored."""
    from paper_2210_08494_b200 import binding
    src = open(os.path.join(ROOT, "include", "bkfac.h")).read()
    defs = {m.group(1): int(m.group(2), 0)
            for m in re.finditer(r"^#define\s+(BKFAC_[A-Z0-9_]+)\s+(0x[0-9a-fA-F]+|\d+)\s*$", src, flags=re.M)}
    opts = [n for n in defs if n.startswith("BKFAC_OPT_")]
    assert len(opts) >= 13 and len(set(defs[n] for n in opts)) == len(opts)
    for n in opts:
        assert hasattr(binding, n), f"binding lacks {n}"
    for n, v in defs.items():
        if hasattr(binding, n):
            assert getattr(binding, n) == v, n


def test_status_strings(lib):
    from paper_2210_08494_b200 import binding
    assert binding.bkfac_status_string(0) == "ok"
    assert binding.bkfac_status_string(4) == "output aliases input"


def test_init_validates_shapes_without_gpu(lib):
    from paper_2210_08494_b200 import binding
    h = ctypes.c_void_p()
    bad = (binding.FactorDesc * 1)(binding.FactorDesc(10, 11, 4, 0))   # r > n
    ld = (binding.LayerDesc * 1)()
    assert lib.bkfac_init(ctypes.byref(h), bad, 1, ld, 0, 0) == 2
    bad = (binding.FactorDesc * 1)(binding.FactorDesc(10, 0, 4, 0))    # r = 0
    assert lib.bkfac_init(ctypes.byref(h), bad, 1, ld, 0, 0) == 2
    assert lib.bkfac_init(None, bad, 1, ld, 0, 0) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2210_08494_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "bkfac_oracle" not in txt, f


def test_shard_layers_lpt():
    from paper_2210_08494_b200.stack import layer_cost, shard_layers
    import synth
    cfg = synth.cfg5_transformer()
    costs = [layer_cost(cfg.factors[l.a_index].n, cfg.factors[l.g_index].n) for l in cfg.layers]
    for w in (1, 2, 4, 8):
        owned = shard_layers(costs, w)
        assert sorted(sum(owned, [])) == list(range(len(costs)))
        assert {len(o) for o in owned} == {48 // w}      # exactly balanced
    cfg3 = synth.cfg3_vgg()
    costs = [layer_cost(cfg3.factors[l.a_index].n, cfg3.factors[l.g_index].n) for l in cfg3.layers]
    owned = shard_layers(costs, 4)
    loads = [sum(costs[i] for i in o) for o in owned]
    # list-scheduling bound: makespan <= total/w + (1 - 1/w) max cost
    assert max(loads) <= sum(costs) / 4 + 0.75 * max(costs) + 1e-6
