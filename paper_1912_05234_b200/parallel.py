"""Data-parallel training across GPUs (one process per GPU, torch.distributed for the plumbing).

The reference parallelises net::train over the examples of each SGD group with a static ceil-block
split (runtime::parallel_build / static_chunk, runtime.cpp:138-191) and then reduces the per-example
gradient cells in example order (network.cpp:236-243).  Across GPUs the same split becomes: rank r
owns static_chunk(m, world, r) of every group, computes its shard's gradient sum on device
(tlb_train_shard_device), one allreduce(sum) of the 3,898-float buffer crosses NVLink (NCCL), and every
rank applies the identical sgd_step with the GLOBAL group size m (network.cpp:244).  The fp64 loss sum
is kept per rank and reduced once per epoch.

The host logic (grouping, sharding, collective, update) lives in ``train_epoch`` with a pluggable
compute backend so it is exercised on CPU with gloo in tests/test_parallel.py.
"""
from __future__ import annotations

from typing import Callable, Protocol

import torch
import torch.distributed as dist

NPARAM, PSTRIDE = 3898, 3904


def static_chunk(n: int, workers: int, w: int) -> tuple[int, int]:
    """runtime::static_chunk (runtime.cpp:138-145): ceil-block split of [0, n)."""
    if n < 0 or workers < 1 or w < 0 or w >= workers:
        raise ValueError("static_chunk: invalid arguments")
    block = (n + workers - 1) // workers
    lo = min(w * block, n)
    return lo, min(lo + block, n)


def groups(n: int, batch: int) -> list[tuple[int, int]]:
    """mnist::batches (mnist.cpp:169-185): consecutive groups [start, start+m) in dataset order."""
    if batch < 1:
        raise ValueError(f"batches: size must be >= 1, got {batch}")
    return [(s, min(batch, n - s)) for s in range(0, n, batch)]


class ShardBackend(Protocol):
    def shard_grad(self, group: int, lo: int, hi: int, grad: torch.Tensor, loss: torch.Tensor) -> None:
        """grad[:3898] = sum of the shard's gradient rows; loss[0] = fp64 sum of its losses."""

    def apply(self, grad: torch.Tensor, rate: float, m: int) -> None:
        """params -= rate * (grad / m)."""


def train_epoch(backend: ShardBackend, n: int, batch: int, rate: float, grad: torch.Tensor,
                loss: torch.Tensor, loss_acc: torch.Tensor, world: int, rank: int,
                allreduce: Callable[[torch.Tensor], None]) -> None:
    """One epoch of data-parallel net::train.  loss_acc (fp64, 1 element) accumulates this rank's
    loss; the caller reduces it across ranks once per epoch."""
    for g, (_, m) in enumerate(groups(n, batch)):
        lo, hi = static_chunk(m, world, rank)
        backend.shard_grad(g, lo, hi, grad, loss)
        loss_acc += loss
        allreduce(grad)
        backend.apply(grad, rate, m)


class DeviceBackend:
    """Shard compute on the B200 through the C ABI (tlb_train_shard_device / tlb_apply_sgd_device)."""

    def __init__(self, ctx, d_images: torch.Tensor, d_labels: torch.Tensor, n: int, batch: int,
                 d_params: torch.Tensor):
        self.ctx, self.x, self.y, self.n, self.batch, self.p = ctx, d_images, d_labels, n, batch, d_params

    def shard_grad(self, group, lo, hi, grad, loss):
        self.ctx.train_shard_device(self.x.data_ptr(), self.y.data_ptr(), self.n, self.batch, group, lo, hi,
                                    self.p.data_ptr(), grad.data_ptr(), loss.data_ptr())

    def apply(self, grad, rate, m):
        self.ctx.apply_sgd_device(self.p.data_ptr(), grad.data_ptr(), rate, m)


class DeviceShardStep:
    """bench.py's N>1 step: weak scaling, one epoch per call, NCCL allreduce per group.

    With ``graph=True`` the epoch (per group: shard kernel, loss add, NCCL allreduce, sgd kernel; then the
    loss allreduce) is captured once into a CUDA graph on the context stream and replayed per epoch, so
    the ~400 launches + collectives of an epoch cost one graph launch on the host.  The parameter and
    epoch-loss buffers are fixed per instance (captured by address)."""

    def __init__(self, ctx, d_images, d_labels, n: int, global_batch: int, world: int, rank: int,
                 graph: bool = False):
        self.ctx, self.x, self.y, self.n, self.B = ctx, d_images, d_labels, n, global_batch
        self.world, self.rank = world, rank
        dev = d_images.device
        self.grad = torch.zeros(PSTRIDE, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.loss_acc = torch.zeros(1, dtype=torch.float64, device=dev)
        self.groups_per_epoch = len(groups(n, global_batch))
        self.use_graph = graph
        self.graph = None
        self.graph_key = None

    def _epoch_body(self, d_params, rate: float, out) -> None:
        backend = DeviceBackend(self.ctx, self.x, self.y, self.n, self.B, d_params)
        self.loss_acc.zero_()
        train_epoch(backend, self.n, self.B, rate, self.grad, self.loss, self.loss_acc, self.world, self.rank,
                    lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM))
        dist.all_reduce(self.loss_acc, op=dist.ReduceOp.SUM)
        out.copy_(self.loss_acc / self.n)

    def epoch(self, d_params, rate: float, d_epoch_loss, e: int) -> None:
        if not self.use_graph:
            self._epoch_body(d_params, rate, d_epoch_loss[e : e + 1])
            return
        key = (d_params.data_ptr(), rate)
        if self.graph is None or self.graph_key != key:
            self.out = torch.zeros(1, dtype=torch.float64, device=self.grad.device)
            self._epoch_body(d_params, rate, self.out)  # eager warm-up: workspaces and communicators exist
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
                self._epoch_body(d_params, rate, self.out)
            # the warm-up ran a real epoch: this instance's callers re-initialise the parameters after
            # warm-up (bench.py resets them), so no correction is applied here
            self.graph, self.graph_key = g, key
        self.graph.replay()
        d_epoch_loss[e : e + 1].copy_(self.out)


class FusedDPStep:
    """Fused data parallelism over NVLink (tlb_train_dp_device): one persistent clustered launch per
    epoch per rank and NO collective call on the data path -- each rank's clusters add their fixed-point
    gradient slices straight into the owning rank's accumulator (slice s on rank s % world) through
    peer pointers of a torch symmetric-memory workspace, wait on that slice's arrival counter, and apply
    the identical update.  Falls back (raises) when symmetric memory is unavailable; a peer that never
    arrives trips the kernel's watchdog (``check()`` raises) instead of hanging."""

    def __init__(self, ctx, d_images, d_labels, n: int, global_batch: int, world: int, rank: int,
                 timeout_s: float = 2.0, ipc: bool = False):
        from . import _lib
        self.ctx, self.x, self.y, self.n, self.B = ctx, d_images, d_labels, n, global_batch
        self.world, self.rank, self.timeout_s = world, rank, timeout_s
        nbytes = int(_lib.lib().tlb_dp_workspace_bytes())
        if not ipc:
            import torch.distributed._symmetric_memory as symm_mem
            self.ws = symm_mem.empty(nbytes, dtype=torch.uint8, device=d_images.device)
            self.ws.zero_()
            group = dist.group.WORLD
            self.handle = symm_mem.rendezvous(self.ws, group.group_name if hasattr(group, "group_name") else group)
            self.peers = [int(p) for p in self.handle.buffer_ptrs]
        else:
            # Plain CUDA IPC handles exchanged over the process group (any backend): the ranks may share
            # one device, which torch symmetric memory refuses -- used to run the cross-process protocol
            # on a single GPU.
            from torch.multiprocessing.reductions import reduce_tensor
            self.ws = torch.zeros(nbytes, dtype=torch.uint8, device=d_images.device)
            torch.cuda.synchronize()
            handles = [None] * world
            dist.all_gather_object(handles, reduce_tensor(self.ws))
            self._peer_tensors = [self.ws if r == rank else fn(*args) for r, (fn, args) in enumerate(handles)]
            self.peers = [int(t.data_ptr()) for t in self._peer_tensors]
        self.err_off = nbytes - 32
        self.seq = 0
        self.groups_per_epoch = len(groups(n, global_batch))
        torch.cuda.synchronize()
        dist.barrier()

    def epoch(self, d_params, rate: float, d_epoch_loss, e: int) -> None:
        self.ctx.train_dp_device(self.x.data_ptr(), self.y.data_ptr(), self.n, d_params.data_ptr(), rate, e, 1, self.B,
                                 d_epoch_loss.data_ptr(), self.world, self.rank, self.peers, self.seq, self.timeout_s)
        self.seq += self.groups_per_epoch

    def check(self) -> None:
        """Raise if a peer wait timed out in any launch so far (reads this rank's watchdog word)."""
        flag = self.ws[self.err_off:self.err_off + 4].view(torch.int32).item()
        if flag:
            raise RuntimeError("fused data parallelism: a peer GPU never arrived (watchdog)")
