"""Host logic of the f2 PRM pass, without a GPU: the packing plan that
lays every row's new suffix entries back to back into chunks (sart_debug_prm_plan, the
function the engine runs at each boundary).  Checked against the plain definition of what
the pass must read (reading R42: row r reads entries ell_ws[r] .. ell[r]-1, each exactly
once, a row's entries in order even across chunks) and the invariants the kernels rely on
(chunk sizes, query blocks inside one segment, the gather at each row's last entry)."""
import numpy as np
import pytest

from paper_2505_13326_b200.sart import debug_prm_plan


def check_plan(ell_ws, ell, chunk, qp):
    seg, qb, gat, ch = debug_prm_plan(ell_ws, ell, chunk, qp)
    n = len(ell_ws)
    total = int(np.sum(np.asarray(ell) - np.asarray(ell_ws)))
    # chunk sizes: full except the last; segment / q-block / gather counts add up
    assert ch[:, 0].sum() == total
    assert all(t == chunk for t in ch[:-1, 0]) and (len(ch) == 0 or 0 < ch[-1, 0] <= chunk)
    assert ch[:, 1].sum() == len(seg) and ch[:, 2].sum() == len(qb) and ch[:, 3].sum() == len(gat)
    # walk the chunks: segments tile each chunk's tokens in order; coverage of (row, entry)
    read = []
    tok_of = {}                                   # (row, entry) -> (chunk, token)
    si = qi = 0
    for c, (ntok, nseg, nqb, ngat) in enumerate(ch):
        pos = 0
        for s in seg[si:si + nseg]:
            t0, cnt, r, e0 = map(int, s)
            assert t0 == pos and cnt > 0
            for j in range(cnt):
                read.append((r, e0 + j))
                tok_of[(r, e0 + j)] = (c, t0 + j)
            pos += cnt
        assert pos == ntok
        # query blocks: consecutive, <= qp, each inside one segment, entries consistent
        for b in qb[qi:qi + nqb]:
            t0, cnt, r, e0 = map(int, b)
            assert 0 < cnt <= qp
            for j in range(cnt):
                assert tok_of[(r, e0 + j)] == (c, t0 + j)
        covered = sorted(t for b in qb[qi:qi + nqb] for t in range(b[0], b[0] + b[1]))
        assert covered == list(range(ntok))
        si += nseg
        qi += nqb
    expect = [(r, e) for r in range(n) for e in range(ell_ws[r], ell[r])]
    assert read == expect                         # every entry once, rows and entries in order
    # gathers: one per row with new entries, at the token of its last entry
    gi = 0
    for c, (ntok, nseg, nqb, ngat) in enumerate(ch):
        for g in gat[gi:gi + ngat]:
            r, t = int(g[0]), int(g[1])
            assert tok_of[(r, int(ell[r]) - 1)] == (c, t)
        gi += ngat
    assert sorted(int(g[0]) for g in gat) == [r for r in range(n) if ell[r] > ell_ws[r]]


@pytest.mark.parametrize("chunk,qp", [(8192, 16), (100, 32), (64, 64), (128, 16), (7, 16), (1, 64)])
@pytest.mark.parametrize("seed", range(4))
def test_prm_plan_random(chunk, qp, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    T = int(rng.integers(1, 500))
    ws = rng.integers(0, 4000, n)
    cnt = rng.integers(0, T + 1, n)
    cnt[rng.random(n) < 0.2] = T                 # many rows ran the whole window
    check_plan(ws, ws + cnt, chunk, qp)


def test_prm_plan_edge_cases():
    check_plan([0], [1], 8192, 16)               # one entry (EOS at the first step)
    check_plan([5, 0, 9], [5, 0, 9], 64, 16)     # no new entries at all
    check_plan([0, 3], [400, 3 + 400], 400, 64)  # rows exactly fill chunks
    check_plan([0, 0, 0], [130, 1, 129], 128, 32)  # a row longer than a chunk, then short rows
