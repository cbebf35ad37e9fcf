"""Bit-plane primitives against a numpy restatement of Appendix B
(bit i of word i/32; whole-view sync stuck cell = first 0 ascending; transfer ranges =
maximal 0-runs ascending; view check = leq of the abstract pair against every cell):
random planes, ragged ranges sharing edge words, empty ranges, several planes per call,
ranges up to 2^24 cells.  Bit-exact."""
import numpy as np
import pytest

from paper_1910_11110_b200.bitmap import RANGE_DTYPE

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def bits_of(words: np.ndarray) -> np.ndarray:
    return np.unpackbits(words.view(np.uint8), bitorder="little")


def words_of(bits: np.ndarray) -> np.ndarray:
    return np.packbits(bits.astype(np.uint8), bitorder="little").view(np.uint32)


def random_planes(rng, n_planes, n_cells, density):
    n_words = n_cells // 32
    bits = (rng.random(n_planes * n_cells) < density).astype(np.uint8)
    # runs: flip long stretches so runs of every length occur
    for _ in range(n_planes * 4):
        a = int(rng.integers(0, n_planes * n_cells))
        bits[a: a + int(rng.integers(1, 5000))] = rng.integers(0, 2)
    return bits, n_words


def random_ranges(rng, n_planes, n_cells, n_words, k):
    r = np.zeros(k, RANGE_DTYPE)
    p = rng.integers(0, n_planes, k)
    lo = rng.integers(0, n_cells, k)
    hi = np.minimum(lo + rng.integers(0, n_cells, k) // rng.integers(1, 64, k), n_cells - 1)
    r["word_off"], r["lo"], r["hi"] = p * n_words, lo, hi
    r["lo"][:3] = [0, 5, 9]
    r["hi"][:3] = [n_cells - 1, 4, 9]  # whole plane, empty, single cell
    return r


def cells(r, n_cells):
    base = int(r["word_off"]) * 32
    return base + int(r["lo"]), base + int(r["hi"])


@pytest.mark.parametrize("n_cells,n_planes,k", [(1 << 12, 5, 200), (1 << 16, 3, 400), (1 << 24, 2, 40), (1 << 14, 4, 3000)])
def test_first_zero_runs_view_check(ctx, n_cells, n_planes, k):
    from paper_1910_11110_b200.bitmap import first_zero, view_check, zero_runs
    rng = np.random.default_rng(n_cells + k)
    bits, n_words = random_planes(rng, n_planes, n_cells, 0.97)
    rbits, _ = random_planes(rng, n_planes, n_cells, 0.5)
    L = torch.from_numpy(words_of(bits).view(np.int32).copy()).cuda()
    R = torch.from_numpy(words_of(rbits).view(np.int32).copy()).cuda()
    ranges = random_ranges(rng, n_planes, n_cells, n_words, k)
    fz = first_zero(ctx, L, ranges)
    off, st, en = zero_runs(ctx, L, ranges, cap=1 << 22)
    ab = rng.integers(0, 4, k).astype(np.uint8)
    ok = view_check(ctx, L, R, ranges, ab)
    for j, r in enumerate(ranges):
        a, b = cells(r, n_cells)
        seg = bits[a: b + 1] if b >= a else bits[:0]
        z = np.nonzero(seg == 0)[0]
        assert fz[j] == (int(r["lo"]) + int(z[0]) if len(z) else 0xFFFFFFFF), j
        # maximal zero runs, ascending, plane-relative cell indices
        d = np.diff(np.concatenate([[1], seg, [1]]).astype(np.int8))
        ws, we = np.nonzero(d == -1)[0], np.nonzero(d == 1)[0] - 1
        o0, o1 = int(off[j]), int(off[j + 1])
        assert o1 - o0 == len(ws), j
        assert np.array_equal(st[o0:o1], ws + int(r["lo"])) and np.array_equal(en[o0:o1], we + int(r["lo"])), j
        rseg = rbits[a: b + 1] if b >= a else rbits[:0]
        want = {1: bool(seg.all()), 2: bool(rseg.all()), 3: bool(seg.all() and rseg.all()),
                0: not bool((seg | rseg).any())}[int(ab[j])]
        assert ok[j] == want, (j, ab[j])


@pytest.mark.parametrize("k", [300, 2500])  # range prefix in each block / a separate scan
def test_range_set_clear(ctx, k):
    from paper_1910_11110_b200.bitmap import range_set
    rng = np.random.default_rng(5 + k)
    n_cells, n_planes = 1 << 18, 4
    bits, n_words = random_planes(rng, n_planes, n_cells, 0.5)
    dev = torch.from_numpy(words_of(bits).view(np.int32).copy()).cuda()
    want = bits.copy()
    for value in (True, False, True):
        ranges = random_ranges(rng, n_planes, n_cells, n_words, k)
        range_set(ctx, dev, ranges, value)
        for r in ranges:
            a, b = cells(r, n_cells)
            if b >= a:
                want[a: b + 1] = 1 if value else 0
        torch.cuda.synchronize()
        assert np.array_equal(bits_of(dev.cpu().numpy().view(np.uint32)), want)


def ref_runs(bits, ranges, n_cells):
    off, st, en = [0], [], []
    for r in ranges:
        a, b = cells(r, n_cells)
        seg = bits[a: b + 1] if b >= a else bits[:0]
        d = np.diff(np.concatenate([[1], seg, [1]]).astype(np.int8))
        st.append(np.nonzero(d == -1)[0] + int(r["lo"]))
        en.append(np.nonzero(d == 1)[0] - 1 + int(r["lo"]))
        off.append(off[-1] + len(st[-1]))
    return np.array(off, np.uint64), np.concatenate(st).astype(np.uint32), np.concatenate(en).astype(np.uint32)


@pytest.mark.parametrize("pattern", ["sparse", "medium", "dense", "mixed"])
def test_zero_runs_staging(ctx, pattern):
    """Zero runs on 2^22-cell planes whose chunks hold few runs (staged once and copied),
    hundreds (staged, copied eight loads per lane at a time), many runs (over the per-chunk
    staging capacity: the chunk is walked again) or both,
    with whole-plane, ragged and empty ranges; plus output truncated at `cap`."""
    from paper_1910_11110_b200.bitmap import zero_runs
    rng = np.random.default_rng({"sparse": 1, "dense": 2, "mixed": 3, "medium": 4}[pattern])
    n_cells, n_planes = 1 << 22, 4
    n = n_planes * n_cells
    if pattern == "sparse":
        bits = (rng.random(n) < 0.99995).astype(np.uint8)
    elif pattern == "dense":
        bits = (rng.random(n) < 0.5).astype(np.uint8)
    elif pattern == "medium":  # ~2.7M runs: several hundred per warp chunk, under its staging cap
        bits = (rng.random(n) < 0.8).astype(np.uint8)
    else:  # dense and sparse stretches alternate
        bits = np.ones(n, np.uint8)
        for a in range(0, n, 1 << 18):
            if rng.random() < 0.5:
                bits[a: a + (1 << 18)] = rng.random(1 << 18) < 0.4
            else:
                bits[a: a + (1 << 18)] = rng.random(1 << 18) < 0.9999
    ranges = random_ranges(rng, n_planes, n_cells, n_cells // 32, 24)
    ranges["word_off"][:n_planes] = np.arange(n_planes) * (n_cells // 32)
    ranges["lo"][:n_planes], ranges["hi"][:n_planes] = 0, n_cells - 1
    ranges["lo"][n_planes], ranges["hi"][n_planes] = 7, 3  # empty
    dev = torch.from_numpy(words_of(bits).view(np.int32).copy()).cuda()
    want_off, want_st, want_en = ref_runs(bits, ranges, n_cells)
    off, st, en = zero_runs(ctx, dev, ranges, cap=len(want_st) + 5)
    assert np.array_equal(off, want_off)
    assert np.array_equal(st, want_st) and np.array_equal(en, want_en)
    cap = max(1, len(want_st) // 3)
    off, st, en = zero_runs(ctx, dev, ranges, cap=cap)
    assert np.array_equal(off, want_off)
    assert np.array_equal(st, want_st[:cap]) and np.array_equal(en, want_en[:cap])


def _ref_sync_cases(frag_log2, n_progs=12, n=1 << 14):
    """(L, R, view range, site, sync runs or stuck cell) for whole-view syncs the reference
    ran: for each generated element program, the longest prefix the reference completes
    (Done), then one extra call R@site on view v with an empty body, whose guard is the
    whole-view sync of v (site Remote: `push v`, needs L, sets R; Local: `pull v`, needs R,
    sets L; elem_host.cpp closure/guard, ast.hpp:144)."""
    import oracle_ffi as o
    from paper_1910_11110_b200.elem import Program
    out = []
    for pid in range(n_progs):
        g = Program.generate(51, pid, n, 8, 6, 0 if pid % 2 else 300, frag_log2=frag_log2)
        calls = []
        for i in range(g.n_calls):
            c = g.calls[i]
            calls.append((c.view, c.kind, c.site, [(c.body[k].effect, c.body[k].site, c.body[k].lo, c.body[k].hi)
                                                  for k in range(c.n_body)]))
        mk = lambda cs: Program(n, g.view_lo, g.view_hi, cs, frag_log2=frag_log2, frag_seed=g.frag_seed)
        rc, r0, L0, R0, _, _, runs0 = o.elem_run("ref", mk(calls), 1 << 16)
        assert rc == 0
        if r0.status != 0:  # keep the prefix before the call that stopped it
            calls = calls[: r0.stuck_call]
            rc, r0, L0, R0, _, _, runs0 = o.elem_run("ref", mk(calls), 1 << 16)
            assert rc == 0 and r0.status == 0
        for v in range(len(g.view_lo)):
            for site in (0, 1):
                rc, r1, _, _, _, _, runs1 = o.elem_run("ref", mk(calls + [(v, 0, site, [])]), 1 << 16)
                assert rc == 0
                rng = (int(g.view_lo[v]), int(g.view_hi[v]))
                if r1.status == 1 and r1.stuck_call == len(calls) and not (r1.stuck_flags & 2):
                    out.append((L0, R0, rng, site, None, r1.stuck_index))
                elif r1.status == 0 and r1.transfers == r0.transfers + 1:
                    out.append((L0, R0, rng, site, runs1[len(runs0):], None))
    return out


@pytest.mark.parametrize("frag_log2", [8, 1])
def test_zero_runs_equal_reference_sync_deltas(ctx, frag_log2):
    """The primitives against syncs the reference itself ran (its own run_annotated over
    its std::map store, from a pre-fragmented start): the transfer ranges of each sync
    (maximal runs of its delta, semantics.hpp:155-166) equal coh_bitmap_extract_zero_runs
    over the view on the destination plane, and a stuck sync names the cell
    coh_bitmap_first_zero finds on the source plane (the first cell that fails, ascending)."""
    import oracle_ffi as o
    from paper_1910_11110_b200.bitmap import first_zero, zero_runs
    if not o.have_ref():
        pytest.skip("oracle/_ref not built")
    cases = _ref_sync_cases(frag_log2)
    n_runs = n_stuck = 0
    for L0, R0, (lo, hi), site, runs, stuck in cases:
        src, dst = (L0, R0) if site else (R0, L0)
        ranges = np.zeros(1, RANGE_DTYPE)
        ranges["word_off"], ranges["lo"], ranges["hi"] = 0, lo, hi
        fz = int(first_zero(ctx, torch.from_numpy(src.view(np.int32).copy()).cuda(), ranges)[0])
        if stuck is not None:
            assert fz == stuck
            n_stuck += 1
            continue
        assert fz == 0xFFFFFFFF
        off, st, en = zero_runs(ctx, torch.from_numpy(dst.view(np.int32).copy()).cuda(), ranges, cap=1 << 16)
        m = int(off[-1])
        got = np.stack([st[:m], en[:m]], axis=1).astype(np.uint32)
        assert np.array_equal(got, runs), (lo, hi, site)
        n_runs += 1
    assert n_runs >= 40 and n_stuck >= 2, (n_runs, n_stuck)
