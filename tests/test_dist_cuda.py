"""The multi-GPU exchange path of paper_1308_2166_b200/dist.py on ONE GPU: a world-size-1 NCCL process
group with the collective path forced on, so the double-buffered broadcast (its own stream, events
ordering it against the engine stream) and the host-fed slice + all-gather run for real.  States must
equal the oracle's bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from gpu_common import assert_states_equal, oracle_run  # noqa: E402
from synth import rmat  # noqa: E402


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("host_feed", [False, True])
def test_exchange_path_one_gpu(pg, host_feed):
    from paper_1308_2166_b200.dist import ShardedCounter
    s = rmat(12, 16, 31)
    r, w = 3000, 2048
    sc = ShardedCounter(r, 6, w, force_exchange=True)
    sc.engine.set_async(True)
    dev = torch.from_numpy(s.view(np.int32)).cuda()
    host = torch.from_numpy(s.view(np.int32)).pin_memory()
    for k in range(0, len(s), w):
        n = min(w, len(s) - k)
        if host_feed:
            sc.push_batch_host(host[k:k + n])
        else:
            sc.push_batch(dev[k:k + n], w=n)
    assert sc.engine.sync() == 0
    o = oracle_run(s, r, 6, w)
    assert_states_equal(sc.engine.state(), o.state(), f"exchange host_feed={host_feed}")
    assert sc.closed_sum() == o.closed_sum() and sc.estimate() == o.estimate()
