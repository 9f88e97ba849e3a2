"""Data-parallel training over NCCL (one process per GPU), SURVEY §8e.

The reference is single-process; this adds the one
exchange step the path needs.  Samples are independent in every hot-path op, so
rank r trains on samples [r*B, (r+1)*B) of the global batch; three couplings
cross the batch and are handled as follows:

  1. masked-CE normalisation by the GLOBAL mask count (nn.py:73-77): every rank
     draws the whole global mask by Philox skip-ahead (a 1.2 MB kernel) and uses
     its count — no collective needed for it;
  2. MaskGIT masks: rank r draws only its shard with counter skip-ahead, so the
     union over ranks is bit-identical to the single-process mask;
  3. parameter gradients: an fp32 SUM all-reduce over NCCL, bucketed per ST block
     in backward order on a dedicated stream so each bucket's transfer overlaps the
     backward of the blocks below it; the optimizer waits on the last bucket.

With the loss already divided by the global count, the summed gradient equals
the single-process gradient of the global batch.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def init_from_env(backend: str | None = None) -> tuple[int, int, int]:
    """torchrun env -> (rank, world, device index); initialises the process group once.

    One process per GPU over NCCL.  When there are more ranks than visible GPUs (JZ_DP_SHARED_GPU=1,
    or world > device count) the ranks share devices round-robin and talk over gloo: NCCL refuses
    two ranks on one device, gloo all-reduces CUDA tensors through host memory.  That mode exists to
    run the multi-process step end to end on a single-GPU box; it is not a performance mode."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local
    if torch.cuda.is_available():
        n = torch.cuda.device_count()
        shared = os.environ.get("JZ_DP_SHARED_GPU", "0") == "1" or world > n
        if shared:
            dev = local % n
            backend = backend or "gloo"
        torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend=backend)
    return rank, world, dev


def shard(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """(b0, b_local) of rank's contiguous slice of the global batch."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by world size {world}")
    per = global_batch // world
    return rank * per, per


def block_buckets(offsets: dict, prefix: str, blocks: int, total: int) -> list[tuple[str, int, int]]:
    """Contiguous gradient ranges in backward-completion order:
    head (params after the last block), block[n-1] .. block[0], embeddings (params before block 0).

    `offsets`: name -> (offset, shape) of contiguous params, or a ParamStore's `extents`
    (name -> (first, end) storage range, which also covers grouped strided views)."""
    def span(v):
        a, b = v
        return (a, b) if isinstance(b, int) else (a, a + max(1, _numel(b)))

    def rng_of(pred):
        idx = [span(v) for n, v in offsets.items() if pred(n)]
        return (min(a for a, _ in idx), max(b for _, b in idx)) if idx else None

    out = []
    first_block = rng_of(lambda n: n.startswith(f"{prefix}.block0."))
    last_block = rng_of(lambda n: n.startswith(f"{prefix}.block{blocks - 1}."))
    if last_block and last_block[1] < total:
        out.append(("head", last_block[1], total))
    for i in reversed(range(blocks)):
        r = rng_of(lambda n, i=i: n.startswith(f"{prefix}.block{i}."))
        out.append((f"block{i}", r[0], r[1]))
    if first_block and first_block[0] > 0:
        out.append(("embed", 0, first_block[0]))
    return out


def _numel(shp) -> int:
    n = 1
    for s in shp:
        n *= s
    return n


class GradAllReduce:
    """Bucketed, stream-overlapped SUM all-reduce of a flat fp32 gradient buffer."""

    def __init__(self, grad_flat: torch.Tensor, buckets: list[tuple[str, int, int]], group=None):
        self.grad = grad_flat
        self.buckets = {name: (a, b) for name, a, b in buckets}
        self.order = [name for name, _, _ in buckets]
        self.group = group
        self.cuda = grad_flat.is_cuda
        self.stream = torch.cuda.Stream(device=grad_flat.device) if self.cuda else None
        self.works = []
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def ready(self, name: str) -> None:
        """Launch the all-reduce of bucket `name` once the work queued so far on the current stream is done."""
        if self.world == 1:
            return
        a, b = self.buckets[name]
        seg = self.grad[a:b]
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ev)
                self.works.append(dist.all_reduce(seg, op=dist.ReduceOp.SUM, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(seg, op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def finish(self) -> None:
        """Make the current stream wait for every launched bucket."""
        for w in self.works:
            w.wait()
        self.works.clear()
        if self.cuda and self.world > 1:
            torch.cuda.current_stream().wait_stream(self.stream)
