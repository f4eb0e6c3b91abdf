"""FillBoundary plan: the O(n) planner must emit the reference's tags, in
the reference's order (golden tags from the reference itself, plus the
literal O(n^2) restatement in the oracle)."""

import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1604_03570_b200 import Box, BoxArray, DistributionMapping, Geometry
from paper_1604_03570_b200.fillplan import build_fill_plan_units, shift_candidates, split_tags

GOLD = os.path.join(os.path.dirname(__file__), "golden", "plans.npz")


def rows(tags):
    out = np.empty((len(tags), 17), dtype=np.int64)
    for n, t in enumerate(tags):
        out[n] = [t.dst_unit, *t.dst_box.lo, *t.dst_box.hi, t.src_unit, *t.src_box.lo, *t.src_box.hi, *t.shift]
    return out


def golden_cases():
    z = np.load(GOLD)
    for name in z["names"]:
        name = str(name)
        v = z[name + "/valids"]
        d = z[name + "/domain"]
        yield name, [Box(r[:3], r[3:]) for r in v], Box(d[:3], d[3:]), tuple(bool(p) for p in z[name + "/periodic"]), \
            int(z[name + "/nghost"][0]), z[name + "/tags"], z[name + "/exec"]


@pytest.mark.parametrize("case", list(golden_cases()), ids=lambda c: c[0])
def test_plan_matches_reference_golden(case):
    name, valids, dom, per, ng, gtags, gexec = case
    geom = Geometry(dom, per)
    plan = build_fill_plan_units(valids, geom, ng, grids=valids)
    assert np.array_equal(rows(plan.tags), gtags), name
    assert np.array_equal(rows(plan.exec_tags), gexec), name


def test_oracle_restatement_matches_golden():
    for name, valids, dom, per, ng, gtags, _ in golden_cases():
        if len(valids) > 64:
            continue
        t = orc.ref_fill_tags([(v.lo, v.hi) for v in valids], (dom.lo, dom.hi), per, ng)
        got = np.array([[a, *b[0], *b[1], c, *d[0], *d[1], *s] for a, b, c, d, s in t], dtype=np.int64).reshape(-1, 17)
        assert np.array_equal(got, gtags), name


def test_random_layouts_vs_oracle_restatement():
    rng = np.random.default_rng(1234)
    for _ in range(60):
        hi = tuple(int(v) for v in rng.integers(2, 14, 3))
        dom = Box((0, 0, 0), hi)
        mgs = tuple(int(v) for v in rng.integers(2, 8, 3))
        cands = BoxArray.chop(dom, mgs).boxes
        keep = [b for b in cands if rng.random() < 0.75] or cands[:1]
        per = tuple(bool(v) for v in rng.integers(0, 2, 3))
        ng = int(rng.choice([1, 2, 3, 5]))
        plan = build_fill_plan_units(keep, Geometry(dom, per), ng, grids=keep)
        t = orc.ref_fill_tags([(v.lo, v.hi) for v in keep], (dom.lo, dom.hi), per, ng)
        want = np.array([[a, *b[0], *b[1], c, *d[0], *d[1], *s] for a, b, c, d, s in t], dtype=np.int64).reshape(-1, 17)
        assert np.array_equal(rows(plan.tags), want)


def test_split_tags_halves_big_tags():
    dom = Box((0, 0, 0), (47, 47, 47))
    plan = build_fill_plan_units([dom], Geometry(dom), 2, grids=[dom])
    ex = plan.exec_tags
    assert len(ex) > len(plan.tags)
    assert all(t.dst_box.ncells <= 4096 or max(t.dst_box.extents[1:]) < 2 for t in ex)
    assert sum(t.dst_box.ncells for t in ex) == sum(t.dst_box.ncells for t in plan.tags)


def test_shift_candidates_zero_first():
    s = shift_candidates(Geometry(Box((0, 0, 0), (7, 7, 7))), 1)
    assert s[0] == (0, 0, 0) and len(s) == 27
    s = shift_candidates(Geometry(Box((0, 0, 0), (2, 2, 2))), 4)  # two images per side
    assert len(s) == 125


def test_c2_plan_tag_count_and_c5_scale_build_time():
    import time

    dom = Box((0, 0, 0), (255, 255, 255))
    ba = BoxArray.chop(dom, 64)
    plan = build_fill_plan_units(list(ba), Geometry(dom), 1, grids=list(ba))
    assert len(plan.tags) == 64 * 26
    dom = Box((0, 0, 0), (511, 511, 511))
    ba = BoxArray.chop(dom, 32)  # 4096 boxes, ng 2
    t0 = time.perf_counter()
    plan = build_fill_plan_units(list(ba), Geometry(dom), 2, grids=list(ba))
    assert len(plan.tags) == 4096 * 26
    assert time.perf_counter() - t0 < 60


def test_grid_outside_domain_rejected():
    dom = Box((0, 0, 0), (7, 7, 7))
    with pytest.raises(ValueError):
        build_fill_plan_units([Box((0, 0, 0), (8, 7, 7))], Geometry(dom), 1, grids=[Box((0, 0, 0), (8, 7, 7))])


def test_boxarray_overlap_and_dm():
    BoxArray([Box((0, 0, 0), (3, 7, 7)), Box((4, 0, 0), (7, 7, 7))])
    with pytest.raises(ValueError):
        BoxArray([Box((0, 0, 0), (4, 7, 7)), Box((4, 0, 0), (7, 7, 7))])
    ba = BoxArray.chop(Box((0, 0, 0), (255, 255, 255)), 64)
    dm = DistributionMapping(ba, 8)
    assert [len(dm.boxes_of(r)) for r in range(8)] == [8] * 8
    # contiguous x-fastest runs: rank r owns boxes 8r..8r+7 (two y-rows of one z-layer)
    assert dm.boxes_of(3) == list(range(24, 32))
    dm = DistributionMapping(ba, 3)
    assert [len(dm.boxes_of(r)) for r in range(3)] == [22, 21, 21]
