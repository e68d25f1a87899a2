"""§8f consumers on the GPU: rank/select directories, batched queries, WT -> WM conversion.

Parity is against the reference's own outputs (tests/golden/golden_next.npz,
made by make_golden_next.py running the reference), plus full-size properties:
a converted c2 tree equals the direct matrix build word for word, and batched
access decodes the text.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_next

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1702_07578_b200 as wv  # noqa: E402
from paper_1702_07578_b200.bitvec import AbsentOccurrenceError, RankSelectBitVector  # noqa: E402
from paper_1702_07578_b200.structures import BitVector  # noqa: E402
from paper_1702_07578_b200.support import DeviceDirectory, DeviceSupport  # noqa: E402


def _rs_cases():
    g = golden_next()
    return range(int(g["rs_count"][0]))


@pytest.mark.parametrize("k", list(_rs_cases()))
def test_directory_and_answers_vs_reference(k):
    g = golden_next()
    n = int(g[f"rs{k}_length"][0])
    words = g[f"rs{k}_words"]
    bv = BitVector(n, words.copy())
    if n:
        d = DeviceDirectory(torch.from_numpy(words.view(np.int64)).cuda(), 1, n).host_arrays(0)
        assert np.array_equal(d["super_zeros"], g[f"rs{k}_super_zeros"])
        assert np.array_equal(d["block_zeros"], g[f"rs{k}_block_zeros"])
        assert np.array_equal(d["samples1"], g[f"rs{k}_samples1"])
        assert np.array_equal(d["samples0"], g[f"rs{k}_samples0"])
        assert d["ones"] == int(g[f"rs{k}_ones"][0])
    sup = RankSelectBitVector(bv)
    assert sup.count(1) == int(g[f"rs{k}_ones"][0])
    for i, r in zip(g[f"rs{k}_rank_pos"], g[f"rs{k}_rank1"]):
        assert sup.rank(1, int(i)) == int(r)
        assert sup.rank(0, int(i)) == int(i) - int(r)
    for x in (0, 1):
        for j, p in zip(g[f"rs{k}_sel{x}_j"], g[f"rs{k}_sel{x}"]):
            if p < 0:
                with pytest.raises(AbsentOccurrenceError):
                    sup.select(x, int(j))
            else:
                assert sup.select(x, int(j)) == int(p)


def test_rank_select_argument_errors():
    """Same errors as the reference (test_bitvec.py:118-130)."""
    sup = RankSelectBitVector(BitVector.from_bits([1, 0, 1, 1]))
    with pytest.raises(ValueError):
        sup.rank(2, 1)
    with pytest.raises(IndexError):
        sup.rank(1, 5)
    with pytest.raises(IndexError):
        sup.rank(1, -1)
    with pytest.raises(ValueError):
        sup.select(1, 0)
    with pytest.raises(ValueError):
        sup.select(3, 1)
    assert issubclass(AbsentOccurrenceError, ValueError)


def _q_cases():
    g = golden_next()
    return range(int(g["q_count"][0]))


@pytest.mark.parametrize("ci", list(_q_cases()))
def test_queries_and_conversion_vs_reference(ci):
    g = golden_next()
    sigma = int(g[f"q{ci}_sigma"][0])
    text = g[f"q{ci}_text"]
    n = text.size
    pos, rpos, syms, js = (g[f"q{ci}_{k}"] for k in ("pos", "rpos", "syms", "js"))
    for kind in ("wt", "wm"):
        st = wv.build_structure(text, sigma, kind)
        # host queries (directories built on the GPU)
        assert [st.access(int(i)) for i in pos] == list(g[f"q{ci}_{kind}_access"])
        assert [st.rank(int(c), int(i)) for c, i in zip(syms, rpos)] == list(g[f"q{ci}_{kind}_rank"])
        for c, j, want in zip(syms, js, g[f"q{ci}_{kind}_select"]):
            if want < 0:
                with pytest.raises(AbsentOccurrenceError):
                    st.select(int(c), int(j))
            else:
                assert st.select(int(c), int(j)) == int(want)
        # batched device queries
        ds = st.device_support()
        if n:
            assert ds.access(torch.from_numpy(pos)).cpu().tolist() == list(g[f"q{ci}_{kind}_access"])
        assert ds.rank(torch.from_numpy(syms), torch.from_numpy(rpos)).cpu().tolist() == \
            list(g[f"q{ci}_{kind}_rank"])
        assert ds.select(torch.from_numpy(syms), torch.from_numpy(js)).cpu().tolist() == \
            list(g[f"q{ci}_{kind}_select"])
    # conversion: recovered histogram, start table, converted dump, position map
    wt = wv.build_structure(text, sigma, "wt")
    assert np.array_equal(wv.recover_histogram(wt), g[f"q{ci}_recovered"])
    want = bytes(g[f"q{ci}_conv_dump"])
    assert wv.dump_structure(wv.convert_wt_to_wm(wt)) == want
    assert wv.dump_structure(wv.convert_wt_to_wm(wt, text=text)) == want
    hist = g[f"q{ci}_recovered"]
    assert wv.dump_structure(wv.convert_wt_to_wm(wt, histogram=hist)) == want
    if n:
        m = wv.TreeToMatrixMap(hist, sigma)
        got = [m.map_position(int(a), int(b)) for a, b in zip(g[f"q{ci}_map_level"], g[f"q{ci}_map_pos"])]
        assert got == list(g[f"q{ci}_map"])


def test_conversion_validation():
    """Same errors as the reference (test_wt2wm.py:131-150)."""
    rng = np.random.default_rng(3)
    text = rng.integers(0, 5, 50).astype(np.uint8)
    wt = wv.build_structure(text, 5, "wt")
    wm = wv.build_structure(text, 5, "wm")
    with pytest.raises(TypeError):
        wv.convert_wt_to_wm(wm)
    with pytest.raises(ValueError):
        wv.convert_wt_to_wm(wt, text=text[:-1])
    with pytest.raises(ValueError):
        wv.convert_wt_to_wm(wt, histogram=[10, 10, 10, 10, 9, 1])
    bad = np.bincount(text, minlength=8).astype(np.int64)
    bad[0] += 1
    with pytest.raises(ValueError):
        wv.convert_wt_to_wm(wt, histogram=bad)


def test_device_query_errors():
    rng = np.random.default_rng(4)
    text = rng.integers(0, 7, 100).astype(np.uint8)
    ds = wv.build_structure(text, 7, "wm").device_support()
    with pytest.raises(IndexError):
        ds.access([100])
    with pytest.raises(IndexError):
        ds.rank(1, [101])
    with pytest.raises(ValueError):
        ds.rank(7, [3])
    with pytest.raises(ValueError):
        ds.select(1, [0])


@pytest.mark.parametrize("config", ["c2"])
def test_full_size_conversion_directory_and_decode(config):
    import workloads
    from paper_1702_07578_b200.device import DeviceBuilder
    from paper_1702_07578_b200.wt2wm import convert_levels_device

    cfg = workloads.CONFIGS[config]
    n, sigma = cfg["n"], cfg["sigma"]
    torch.cuda.empty_cache()
    text = workloads.generate(config)
    b = DeviceBuilder()
    wt = b.build(text, sigma, "wt", histogram=True)
    wm_words, zeros = convert_levels_device(wt.level_words, n, sigma, wt.hist.cpu().numpy(), builder=b)
    del wt
    wm = b.build(text, sigma, "wm")
    assert torch.equal(wm_words, wm.level_words)
    assert zeros == [int(z) for z in wm.zeros.cpu().tolist()]
    del wm_words
    ds = DeviceSupport.from_build(wm)
    # directory totals: a matrix level's zeros are its zero count Z[l]
    ones = ds.dir.ones.cpu()
    assert [n - int(o) for o in ones.tolist()] == [int(z) for z in wm.zeros.cpu().tolist()]
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    pos = torch.randint(0, n, (1 << 16,), generator=g, device="cuda", dtype=torch.int64)
    pos[:3] = torch.tensor([0, 1, n - 1], device="cuda")
    want = text[pos].to(torch.int64)
    assert torch.equal(ds.access(pos), want)
    # rank / select consistency on the decoded symbols: select(c, rank(c, i) + 1) == i
    r = ds.rank(want, pos)
    assert torch.equal(ds.select(want, r + 1), pos)
