"""GPU checks of the (batch x K) sharding used when the batch is smaller than
the number of GPUs (SURVEY 8(e) K-split, 8(f) NEXT-3; dist.grid_shard).

Only one GPU is available, so every rank's shard is computed in turn in this
process, exactly as that rank would (its own plan over its samples and its
own kernel slice, its own filter transform); the assembled output must equal
the single-plan output bit for bit (reading #8)."""
import pytest
import torch

import paper_1611_06565_b200 as pkg
from paper_1611_06565_b200.dist import grid_shape, grid_shard
from paper_1611_06565_b200.workloads import CONFIGS, SMALL, make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _full(cfg, x, g):
    p = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, cfg.K, x.shape[0], cfg.padding)
    p.filter_transform(g.cuda())
    y = p.forward(x.cuda()).cpu()
    p.close()
    return y


def _sharded(cfg, x, g, world):
    B = x.shape[0]
    y = torch.full((B, cfg.K) + cfg.out_dims, float("nan"))
    for rank in range(world):
        b0, b1, k0, k1 = grid_shard(B, cfg.K, rank, world)
        p = pkg.Plan(cfg.N, cfg.dims, cfg.m, cfg.r, cfg.C, k1 - k0, b1 - b0, cfg.padding)
        p.filter_transform(g[k0:k1].contiguous().cuda())
        y[b0:b1, k0:k1] = p.forward(x[b0:b1].contiguous().cuda()).cpu()
        p.close()
    return y


@pytest.mark.parametrize("name,B,world", [("c2", 1, 2), ("c2", 2, 6), ("c3", 1, 4), ("c4", 2, 4), ("c5", 1, 8)])
def test_grid_shards_equal_single_plan_bitwise(name, B, world):
    cfg = SMALL[name]
    x, g = make_inputs(cfg)
    x = x[:B].contiguous()
    pb, pk = grid_shape(B, cfg.K, world)
    assert pk > 1                                    # the K split is exercised
    assert torch.equal(_sharded(cfg, x, g, world), _full(cfg, x, g))


def test_c1_batch1_split_over_4():
    # BJ c1: batch 1, K = 4 -> one output channel per rank
    cfg = CONFIGS["c1"]
    x, g = make_inputs(cfg)
    assert grid_shape(1, 4, 4) == (1, 4)
    assert torch.equal(_sharded(cfg, x, g, 4), _full(cfg, x, g))
