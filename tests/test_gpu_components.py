"""Connected components on the device (csrc/sample.cu bitmap_components: the
shared-memory flood fill behind cw_connected_components, k_reach and k_spawn) on
grids the scene fixtures do not produce: widths that are not multiples of 32, one
row / one column, checkerboards (every cell its own 8-neighbour of two diagonals),
many tiny components, a single spiral corridor (one component, many passes), and the
union-find fallback for grids whose bitmaps exceed the shared-memory budget.

Checked against the reference's connected_components (routes.py:14-32, restated in
oracle/crowd.py) for the ids, and against a 4-connected labelling for reach."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle_cc(ok):
    from oracle.crowd import components
    return components(ok)


def _spiral(n):
    g = np.zeros((n, n), dtype=bool)
    r0, c0, r1, c1 = 0, 0, n - 1, n - 1
    while r0 <= r1 and c0 <= c1:
        g[r0, c0:c1 + 1] = True
        g[r0:r1 + 1, c1] = True
        if r1 - r0 >= 2:
            g[r1, c0:c1 + 1] = True
        if c1 - c0 >= 2:
            g[r0 + 2:r1 + 1, c0] = True
        r0, c0, r1, c1 = r0 + 2, c0 + 2, r1 - 2, c1 - 2
        if r0 <= r1:
            g[r0 - 1, c0] = c0 <= c1
    return g


def _cases():
    rng = np.random.default_rng(7)
    cases = {}
    for ny, nx in ((1, 1), (1, 70), (70, 1), (33, 31), (40, 100), (129, 65), (256, 256)):
        for p in (0.3, 0.55, 0.8, 1.0):
            cases[f"rand{ny}x{nx}_{p}"] = rng.random((ny, nx)) < p
    yy, xx = np.mgrid[:64, :96]
    cases["checker"] = (yy + xx) % 2 == 0
    cases["dots"] = (yy % 2 == 0) & (xx % 2 == 0)
    cases["stripes_h"] = yy % 2 == 0
    cases["spiral"] = _spiral(97)
    cases["empty"] = np.zeros((50, 77), dtype=bool)
    return cases


@pytest.mark.parametrize("name", sorted(_cases()))
def test_connected_components_matches_reference(name):
    from paper_2505_00690_b200.crowd import connected_components
    ok = _cases()[name]
    assert np.array_equal(connected_components(ok), _oracle_cc(ok)), name


def test_connected_components_union_find_fallback():
    # 1100 x 1100: the bitmaps exceed the shared-memory budget, the global union-find runs
    from paper_2505_00690_b200.crowd import connected_components
    rng = np.random.default_rng(3)
    ok = rng.random((1100, 1100)) < 0.6
    got = connected_components(ok)
    from scipy import ndimage
    lab, n = ndimage.label(ok, structure=np.ones((3, 3), dtype=int))
    # same partition, ids in row-major order of each component's first cell
    first = np.full(n + 1, -1)
    flat = lab.ravel()
    idx = np.flatnonzero(flat)
    order = np.unique(flat[idx], return_index=True)
    rank = np.argsort(np.argsort(idx[order[1]]))
    first[order[0]] = rank
    want = np.where(ok, first[lab], -1)
    assert np.array_equal(got, want)


def test_reach_is_the_4_connected_partition():
    """k_reach labels of sampled scenes: the 4-connected components of the passable
    cells (labels != OBSTACLE), each labelled by its smallest cell index."""
    import torch
    from scipy import ndimage

    import bench
    from paper_2505_00690_b200.rng import child_seeds_device
    from paper_2505_00690_b200.urbangen import SceneSampler

    saved = dict(bench.CFG)
    for cfg, E in (("cfg2", 16), ("cfg4", 2)):
        bench.CFG.clear()
        bench.CFG.update(bench.CONFIGS[cfg])
        dev = torch.device("cuda")
        es = child_seeds_device(torch.zeros(E, dtype=torch.int64, device=dev), "env", torch.arange(E, device=dev))
        s = SceneSampler(bench.make_spec(), E)
        b = s.sample(es, child_seeds_device(es, "crowd", 0))
        labels = b.labels.cpu().numpy()
        reach = b.reach.cpu().numpy()
        for e in range(E):
            lab = labels[e].reshape(-1)
            ny = int(round(np.sqrt(lab.size)))
            ok = (lab != 0).reshape(ny, -1)
            comp, n = ndimage.label(ok)
            flat = comp.ravel()
            want = np.full(flat.size, -1, dtype=np.int64)
            for k in range(1, n + 1):
                cells = np.flatnonzero(flat == k)
                want[cells] = cells.min()
            assert np.array_equal(reach[e].reshape(-1), want), (cfg, e)
    bench.CFG.clear()
    bench.CFG.update(saved)
