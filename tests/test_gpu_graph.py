"""The perimeter-graph solver (H5; "solved using the same strategy
described in Algorithm 1") both ways: one cooperative persistent
kernel that takes every decision on the device (FA_OPT_GRAPH = device) and
the host-driven kernels (host, the default).  Deep graphs force the chain
contraction and its recursion; cycles must be reported; results equal the
oracle exactly (integers) or within D13 (f64, absorption)."""
import numpy as np
import pytest
import torch

import inputs
import oracle

pytestmark = pytest.mark.gpu


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(params=["device", "host", "auto"])
def graph(request):
    return request.param


def test_graph_serpentine_cfg2(fa_lib, graph):
    d = inputs.serpentine(4096, 4096)
    with fa_lib.Context(0) as ctx:
        ctx.set_option("graph", graph)
        got = ctx.accumulate(dirs=_cuda(d), atype="u32").cpu().numpy()
        st = ctx.stats()
    y, x = np.mgrid[0:4096, 0:4096].astype(np.uint64)
    assert (got == (4096 * y + np.where(y % 2 == 0, x, 4095 - x) + 1)).all()
    assert st["contract_levels"] >= 1  # one 520K-node chain of block exits: contracted


@pytest.mark.parametrize("cap", [0, 1, 4, 128])
def test_graph_walk_caps_random_and_transposed(fa_lib, graph, cap):
    r = inputs.random_dirs(cap + 3, 700, 513, p_nodata=0.1, p_noflow=0.02)
    w = inputs.weights_u32(cap + 3, r.shape, 0, 100)
    t = inputs.serpentine(768, 512, transposed=True)
    with fa_lib.Context(0, tile=(128, 96)) as ctx:
        ctx.set_option("graph", graph)
        ctx.set_option("walk_cap", cap)
        assert (ctx.accumulate(dirs=_cuda(r), w=_cuda(w), atype="u64").cpu().numpy() == oracle.accumulate(r, w)).all()
        assert (ctx.accumulate_strips(3, dirs=_cuda(r), w=_cuda(w), atype="u64").cpu().numpy()
                == oracle.accumulate(r, w)).all()
        got = ctx.accumulate(dirs=_cuda(t), atype="u32").cpu().numpy()
    assert (got == oracle.accumulate(t).astype(np.uint32)).all()


def test_graph_f64_and_absorption(fa_lib, graph):
    cfg = inputs.make_config("cfg3", 1024, 1024)
    d = oracle.d8(cfg.dem)
    rng = np.random.default_rng(7)
    al = (0.999 + 0.001 * rng.random(d.shape)).astype(np.float32)
    s = inputs.serpentine(1024, 1024)
    with fa_lib.Context(0, tile=(256, 256)) as ctx:
        ctx.set_option("graph", graph)
        got = ctx.accumulate(dem=_cuda(cfg.dem), w=_cuda(cfg.w), atype="f64").cpu().numpy()
        ga = ctx.accumulate_absorb(_cuda(al), dirs=_cuda(s)).cpu().numpy()
        gs = ctx.accumulate_absorb(_cuda(al), dirs=_cuda(s), nstrips=4).cpu().numpy()
    data = d != 255
    exp = oracle.accumulate(d, cfg.w, kind="f64")
    assert (np.abs(got[data] - exp[data]) <= 1e-9 * exp[data]).all()
    ea = oracle.accumulate_alpha(s, al)
    assert (np.abs(ga - ea) <= 1e-9 * np.abs(ea)).all()
    assert (np.abs(gs - ea) <= 1e-9 * np.abs(ea)).all()


def test_graph_cycles_reported(fa_lib, graph):
    d = np.zeros((256, 256), np.uint8)
    d[100, 10:200] = 3          # a long loop through many blocks
    d[100:160, 200] = 5
    d[160, 11:201] = 7
    d[101:161, 10] = 1
    d[100, 200], d[160, 200], d[160, 10], d[100, 10] = 5, 7, 1, 3
    with fa_lib.Context(0, tile=(64, 64)) as ctx:
        ctx.set_option("graph", graph)
        for call in (lambda: ctx.accumulate(dirs=_cuda(d)), lambda: ctx.accumulate_strips(2, dirs=_cuda(d))):
            with pytest.raises(fa_lib.FaError) as e:
                call()
            assert e.value.status == fa_lib.FA_E_CYCLE
