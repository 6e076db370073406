"""Multi-GPU plumbing for the RaaS decode path.

Units (request, kv-head) are independent (reading D5), so the path shards with no collective:

* request sharding (the bench's default): rank r owns a contiguous block of requests, with its
  own handles and arenas; NCCL is used only for barriers and the max-over-ranks timing.
* head sharding (for small batches, e.g. config 2 at B = 1): rank r owns a contiguous block of
  kv-heads and their q-heads; the step is the same kernel over this rank's units, followed by
  one all-gather of `out` per layer-step (the only collective of the path).  ``HeadGather``
  preallocates its buffers, so the decode launches and the NCCL all-gathers of a model step
  are captured together in one CUDA graph.

The helpers here are plain index arithmetic and torch.distributed calls; the decode itself is
always libraas on this rank's GPU.
"""
from __future__ import annotations


def request_range(global_batch: int, world: int, rank: int):
    """Contiguous, balanced block of requests [lo, hi) owned by `rank`."""
    if not (0 <= rank < world) or global_batch < 0:
        raise ValueError("bad request shard")
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def head_range(n_kv_heads: int, n_q_heads: int, world: int, rank: int):
    """kv-heads [kv_lo, kv_hi) and q-heads [q_lo, q_hi) owned by `rank` (GQA groups stay whole,
    reading D15: q-head h uses kv-head h // g)."""
    if n_kv_heads % world != 0 or n_q_heads % n_kv_heads != 0:
        raise ValueError("head sharding needs n_kv_heads % world == 0")
    g = n_q_heads // n_kv_heads
    per = n_kv_heads // world
    kv_lo = rank * per
    return kv_lo, kv_lo + per, kv_lo * g, (kv_lo + per) * g


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a scalar (timing: a multi-GPU number is the slowest rank's)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_heads(out_local, out_full=None):
    """All-gather of a head-sharded output.  out_local: [B, Hq/G, d] on this rank; returns
    [B, Hq, d] with rank r's heads at [r*Hq/G, (r+1)*Hq/G).  Uses all_gather_into_tensor on
    NCCL (one NVLink collective), list all_gather elsewhere (gloo tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    B, hl, d = out_local.shape
    if dist.get_backend() == "nccl":
        stacked = torch.empty((world, B, hl, d), dtype=out_local.dtype, device=out_local.device)
        dist.all_gather_into_tensor(stacked, out_local.contiguous())
    else:  # gloo (CPU tests, the bench's shared-GPU test mode): gather on the host
        loc = out_local.contiguous().cpu()
        parts = [torch.empty_like(loc) for _ in range(world)]
        dist.all_gather(parts, loc)
        stacked = torch.stack(parts).to(out_local.device)
    full = stacked.permute(1, 0, 2, 3).reshape(B, world * hl, d)
    if out_full is not None:
        out_full.copy_(full)
        return out_full
    return full


class HeadGather:
    """Preallocated all-gather of a head-sharded output, [B, Hq/G, d] per rank -> [B, Hq, d]
    (rank r's heads at [r*Hq/G, (r+1)*Hq/G)).  Nothing is allocated per call, so a step that
    uses it can be captured in a CUDA graph with NCCL (all_gather_into_tensor is capturable).
    At B = 1 the rank-major gather layout [G][1][Hq/G][d] IS [1][Hq][d]: NCCL writes the final
    tensor directly; for B > 1 one strided copy reorders it.  gloo (CPU tests, the bench's
    shared-GPU test mode) goes through the host and is not capturable."""

    def __init__(self, B, hq_local, d, dtype, device):
        import torch
        import torch.distributed as dist

        self.world = dist.get_world_size()
        self.B, self.hl, self.d = B, hq_local, d
        self.nccl = dist.get_backend() == "nccl"
        self.full = torch.empty((B, self.world * hq_local, d), dtype=dtype, device=device)
        self.stacked = (self.full if B == 1 else
                        torch.empty((self.world, B, hq_local, d), dtype=dtype, device=device))
        self.capturable = self.nccl

    def __call__(self, out_local):
        import torch
        import torch.distributed as dist

        if self.nccl:
            dist.all_gather_into_tensor(self.stacked, out_local)
        else:
            loc = out_local.contiguous().cpu()
            parts = [torch.empty_like(loc) for _ in range(self.world)]
            dist.all_gather(parts, loc)
            self.stacked.copy_(torch.stack(parts).view(self.stacked.shape))
        if self.B > 1:
            self.full.view(self.B, self.world, self.hl, self.d).copy_(self.stacked.permute(1, 0, 2, 3))
        return self.full
