"""Host-side invariants of the fused MLP step's list schedule (brk_mlp.cu mlp_list_schedule):
the grouped launch cannot deadlock only if every CTA pair runs its units in increasing global
order and every dependency points to an earlier problem; every unit must be run exactly once.
No GPU needed (the scheduler is host code)."""

import ctypes

import pytest

from paper_1906_06440_b200 import _lib


def _schedule(L, N, C, pairs):
    fn = _lib.load().brk_diag_mlp_schedule
    units = (ctypes.c_int16 * 2048)()
    offs = (ctypes.c_int16 * 81)()
    tiles = (ctypes.c_int * 16)()
    dep = (ctypes.c_int * 16)()
    n = fn(L, N, C, pairs, units, offs, tiles, dep)
    return n, list(units[:n]), list(offs[:pairs + 1]), list(tiles[:3 * L]), list(dep[:3 * L])


@pytest.mark.parametrize("L,N,C,pairs", [(4, 2048, 1024, 74), (4, 2048, 1024, 72), (2, 256, 256, 74),
                                         (3, 512, 512, 37), (4, 1024, 512, 10), (1, 256, 256, 1)])
def test_list_schedule_is_deadlock_free_and_complete(L, N, C, pairs):
    n, units, offs, tiles, dep = _schedule(L, N, C, pairs)
    assert n == sum(tiles) > 0
    assert offs[0] == 0 and offs[-1] == n
    seen = set()
    for c in range(pairs):
        lst = units[offs[c]:offs[c + 1]]
        assert all(a < b for a, b in zip(lst, lst[1:])), f"pair {c}: units not in global order"
        seen.update(lst)
    assert seen == set(range(n)), "every unit exactly once"
    assert all(d < q for q, d in enumerate(dep)), "dependencies point backwards"
