"""Multi-GPU partition of the text and the two exchange steps.

The text t[0..N) is split into G contiguous shards.  Rank g OWNS the alignments
[a_g, a_{g+1}) with a_g = align16(g * N / G) and HOLDS the bytes
[a_g, min(a_{g+1} + H, N)) -- its owned bytes plus an H-byte halo (H >= m - 1
for every pattern searched).  For a pattern of length m rank g searches the view
t_g = held[0 : min(a_{g+1} + m - 1, N) - a_g]: its alignments are exactly the
owned ones clipped to [0, N - m], so every occurrence is counted by exactly one
rank and the per-rank counts add up to the global count (no overlap, no gap).

Exchanges (torch.distributed over NCCL / NVLink; gloo on CPU in the tests):
  * once per text: all_reduce(SUM) of the owned-byte histograms, so every rank
    derives the same rarest-first order pi as a 1-GPU run (reading R14);
  * per pattern batch: all_reduce(SUM) of the device int64 counts -- or, where the
    platform provides NVLink multicast (torch symmetric memory), no collective at
    all: each rank's counts are added to every rank's copy with multimem.red through
    an NVLink multicast address (count_sharded_fused, NEXT-4).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

ALIGN = 16


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    N: int          # global text length
    own_lo: int     # first owned alignment / first held byte
    own_hi: int     # one past the last owned alignment (= next shard's own_lo)
    halo: int       # H: bytes held past own_hi (clipped at N)

    @property
    def held_hi(self) -> int:
        return min(self.own_hi + self.halo, self.N)

    @property
    def held_len(self) -> int:
        return self.held_hi - self.own_lo

    @property
    def owned_bytes(self) -> int:
        return self.own_hi - self.own_lo

    def view_len(self, m: int) -> int:
        """Length of the local text view that counts exactly the owned alignments for length m."""
        if m - 1 > self.halo and self.own_hi < self.N:
            raise ValueError(f"pattern length {m} needs a halo >= {m - 1}, shard has {self.halo}")
        return max(0, min(self.own_hi + m - 1, self.N) - self.own_lo)


def shard_bounds(N: int, world: int) -> List[int]:
    """a_0 = 0 <= a_1 <= ... <= a_G = N, interior cuts rounded down to 16 bytes."""
    cuts = [0]
    for g in range(1, world):
        c = (g * N // world) // ALIGN * ALIGN
        cuts.append(max(c, cuts[-1]))
    cuts.append(N)
    return cuts


def make_shard(N: int, rank: int, world: int, halo: int) -> Shard:
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    b = shard_bounds(N, world)
    return Shard(rank, world, N, b[rank], b[rank + 1], halo)


def all_shards(N: int, world: int, halo: int) -> List[Shard]:
    return [make_shard(N, g, world, halo) for g in range(world)]


# ----------------------------------------------------------------------------- collectives

def allreduce_sum_(tensor, group=None):
    """In-place SUM all-reduce (no-op when torch.distributed is not initialised or world == 1)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def global_histogram(shard_text, shard: Shard, group=None, stream=None):
    """Histogram of the OWNED bytes of this rank's shard, summed over ranks (device int64[256])."""
    import paper_1612_01506_b200 as sm
    h = sm.sm_histogram(shard_text[: shard.owned_bytes], stream=stream)
    return allreduce_sum_(h, group)


def count_sharded(patterns, shard_text, shard: Shard, hist, counts=None, group=None, stream=None,
                  strategy: int = 0):
    """Global counts of each pattern: batched local launches over the rank's held bytes,
    counting only its owned alignments, + one all_reduce of int64[P]."""
    import torch

    import paper_1612_01506_b200 as sm
    pb = patterns if isinstance(patterns, sm.PatternBatch) else sm.PatternBatch(patterns)
    if counts is None:
        counts = torch.zeros(max(pb.P, 1), dtype=torch.int64, device=shard_text.device)
    max_m = max((len(p) for p in pb.data), default=1)
    shard.view_len(max_m)  # halo check
    held = shard_text[: shard.held_len]
    sm.sm_count_batch(pb, held, counts, hist=hist, max_alignments=shard.owned_bytes, strategy=strategy,
                      stream=stream)
    return allreduce_sum_(counts, group)


class MulticastCounts:
    """NEXT-4: an int64 count buffer in torch symmetric memory whose NVLink multicast
    address sm_count_batch_multicast reduces into (one multimem.red per pattern after the
    search launches: the all-reduce done by the switch, no NCCL call).  `available` is False when the
    platform gives no multicast pointer (e.g. a single-GPU box, where cuMulticastCreate is
    refused); count_sharded_fused then uses count_sharded's NCCL all-reduce instead."""

    def __init__(self, P: int, device, group=None):
        import torch
        import torch.distributed as dist
        self.P, self.group, self.available = P, group, False
        self.local = None
        try:
            import torch.distributed._symmetric_memory as symm_mem
            self.local = symm_mem.empty(max(P, 1), dtype=torch.int64, device=device)
            h = symm_mem.rendezvous(self.local, group if group is not None else dist.group.WORLD)
            self.mc_ptr = int(getattr(h, "multicast_ptr", 0) or 0)
            self.available = self.mc_ptr != 0
        except Exception:
            self.available = False


def count_sharded_fused(patterns, shard_text, shard: Shard, hist, mc: "MulticastCounts", group=None,
                        strategy: int = 0):
    """Global counts with the reduction fused into the kernel when `mc.available`:
    zero the local copy, barrier, one multicast count launch per batch, device sync,
    barrier -> every rank's mc.local holds the global sums.  Else count_sharded."""
    import torch
    import torch.distributed as dist

    import paper_1612_01506_b200 as sm
    if not mc.available:
        return count_sharded(patterns, shard_text, shard, hist, group=group, strategy=strategy)
    pb = patterns if isinstance(patterns, sm.PatternBatch) else sm.PatternBatch(patterns)
    if pb.P > mc.P:
        raise ValueError(f"{pb.P} patterns but the multicast count buffer holds {mc.P}")
    shard.view_len(max((len(p) for p in pb.data), default=1))  # halo check
    mc.local.zero_()
    torch.cuda.synchronize()
    dist.barrier(group=group)
    sm.sm_count_batch_multicast(pb, shard_text[: shard.held_len], mc.mc_ptr, hist=hist,
                                max_alignments=shard.owned_bytes, strategy=strategy)
    torch.cuda.synchronize()
    dist.barrier(group=group)
    return mc.local[: pb.P]


def gather_reports(local_counts, local_pos, group=None):
    """Combine per-rank reports (NEXT-4): every rank passes its int64[P] counts and its
    positions concatenated by pattern (global positions, ascending within a pattern).
    Returns (global counts int64[P], global positions concatenated by pattern) on every
    rank.  Ranks own ascending contiguous alignment ranges, so pattern k's global list
    is rank 0's segment k, then rank 1's, ... (already sorted)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local_counts, local_pos
    world = dist.get_world_size(group)
    P = local_counts.numel()
    counts = [torch.empty_like(local_counts) for _ in range(world)]
    dist.all_gather(counts, local_counts, group=group)
    totals = [int(c.sum().item()) for c in counts]
    width = max(max(totals), 1)
    padded = torch.zeros(width, dtype=local_pos.dtype, device=local_pos.device)
    padded[: local_pos.numel()] = local_pos
    gathered = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(gathered, padded, group=group)
    starts = [torch.cumsum(c, 0) - c for c in counts]  # segment start of pattern k on rank r
    cnt = [c.tolist() for c in counts]
    st = [s.tolist() for s in starts]
    pieces = []
    for k in range(P):
        for r in range(world):
            if cnt[r][k]:
                pieces.append(gathered[r][st[r][k]: st[r][k] + cnt[r][k]])
    pos = torch.cat(pieces) if pieces else local_pos[:0]
    return torch.stack(counts).sum(0), pos


def report_sharded(patterns, shard_text, shard: Shard, hist, group=None, stream=None, strategy: int = 0):
    """Global reports: each rank reports the occurrences at its owned alignments as global
    positions (position_offset = its first owned position), then gather_reports."""
    import torch

    import paper_1612_01506_b200 as sm
    pb = patterns if isinstance(patterns, sm.PatternBatch) else sm.PatternBatch(patterns)
    shard.view_len(max((len(p) for p in pb.data), default=1))  # halo check
    held = shard_text[: shard.held_len]
    counts = torch.zeros(max(pb.P, 1), dtype=torch.int64, device=shard_text.device)[: pb.P]
    sm.sm_report_batch(pb, held, None, counts, hist=hist, max_alignments=shard.owned_bytes, strategy=strategy,
                       stream=stream)  # sizing call (cap 0: counts only)
    total = int(counts.sum().item())
    pos = torch.empty(max(total, 1), dtype=torch.int64, device=shard_text.device)[:total]
    sm.sm_report_batch(pb, held, pos if total else None, counts, hist=hist, max_alignments=shard.owned_bytes,
                       strategy=strategy, stream=stream, position_offset=shard.own_lo)
    return gather_reports(counts, pos, group)
