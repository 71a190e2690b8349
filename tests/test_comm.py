"""Exchange transport on the B200 (-m gpu): sv_comm_bench with a one-rank NCCL communicator sends to
itself through the same grouped ncclSend/ncclRecv + asynchronous-error wait the sharded exchanges use,
and checks every received double against the sender's seeded pattern on the device. (Multi-rank runs:
scripts/comm_bench.py under torchrun; the pool gives one GPU per call.)"""
from __future__ import annotations

import pytest

import paper_2402_08136_b200 as pkg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pattern", [0, 1])
@pytest.mark.parametrize("nbytes", [8 << 10, 256 << 20])
def test_comm_bench_single_rank(pattern, nbytes):
    r = pkg.comm_bench(world=1, pattern=pattern, nbytes=nbytes, reps=3)
    assert r["mismatches"] == 0, r
    assert r["ms"] > 0 and r["gbs"] > 0


def test_comm_bench_rejects_bad_arguments():
    with pytest.raises(pkg.SVError):
        pkg.comm_bench(world=3)
    with pytest.raises(pkg.SVError):
        pkg.comm_bench(world=1, nbytes=12)
    with pytest.raises(pkg.SVError):
        pkg.comm_bench(world=1, pattern=2)
