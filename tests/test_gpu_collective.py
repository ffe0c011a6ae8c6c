"""The token all-gather through the C ABI (dp_allgather_tokens):
a world-1 communicator on the box's one GPU, eager and captured in a CUDA
graph (the bench replays it inside the timed step).  Multi-rank row
ownership and gather order are covered on CPU by test_sharded_cpu.py."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    import build

    build.build()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_allgather_tokens_world1_eager_and_graphed(torch_cuda):
    torch = torch_cuda
    from paper_2512_00719_b200.sharded import BatchShard, NcclTokenGather

    sh = BatchShard(1000, 1, 0)
    g = NcclTokenGather(sh, "cuda:0")
    try:
        local = torch.randint(0, 152064, (1000,), dtype=torch.int32, device="cuda")
        out = torch.full((1000,), -1, dtype=torch.int32, device="cuda")
        g(local, out=out)
        torch.cuda.synchronize()
        assert torch.equal(out, local)
        # captured: the graph replays the collective on new data
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                g(local, out=out)
        torch.cuda.current_stream().wait_stream(s)
        local.copy_(torch.arange(1000, dtype=torch.int32, device="cuda"))
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, local)
    finally:
        g.close()
