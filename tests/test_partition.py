"""Row partition of the sharded mode: qp_partition_rows (host-only C ABI) is
bit-exact against the oracle's plain definition, and the split has the properties the sharded
path relies on (contiguous, covering, monotone, weight-balanced)."""
import numpy as np
import pytest

from oracle.sharded import partition_rows as oracle_partition


def _indptr(row_nnz):
    return np.concatenate([[0], np.cumsum(row_nnz)]).astype(np.int64)


CASES = [
    ("uniform", np.full(300, 4)),
    ("zipf", np.minimum(512, np.random.default_rng(0).zipf(2.1, 5000) + 2)),
    ("empty_rows", np.r_[np.zeros(50, int), np.full(10, 100), np.zeros(50, int)]),
    ("one_heavy", np.r_[np.ones(20, int), [10000], np.ones(20, int)]),
    ("tiny", np.array([3, 1])),
]


@pytest.mark.parametrize("name,row_nnz", CASES)
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_matches_definition(name, row_nnz, world):
    from paper_2104_12916_b200.binding import partition_rows
    m2 = len(row_nnz)
    if world > m2:
        pytest.skip("world > m2 is rejected by qp_setup")
    ip = _indptr(row_nnz)
    lib = partition_rows(ip, m2, world)
    ref = oracle_partition(ip, m2, world)
    assert np.array_equal(lib, ref), (lib, ref)
    assert lib[0] == 0 and lib[-1] == m2 and np.all(np.diff(lib) >= 0)
    w = row_nnz + 1
    total = w.sum()
    heaviest = w.max()
    for r in range(world):
        part = w[lib[r]:lib[r + 1]].sum()
        assert part <= total / world + heaviest + 1e-9      # balanced up to one row
