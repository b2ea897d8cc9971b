"""Multi-GPU partition of the grouped n:m SpMM.

One process per GPU (torchrun), torch.distributed over NCCL for the plumbing.
Tokens are independent columns of B and C, so the product itself needs no
collective:

* token (column) sharding -- the sparse weight (values, idx) is replicated,
  rank p owns columns [c0_p, c1_p) of B and computes C[:, c0_p:c1_p]; an
  all-gather of the C shards follows only when a consumer needs all of C;
* row sharding -- rank p owns whole groups [p*G/P, (p+1)*G/P) of the weight,
  B is replicated, and the all-gather runs along M (contiguous rows of C).

Every rank uses the plan of the GLOBAL problem (sten_spmm_plan_query on the
full shape), so the per-column summation order equals the single-GPU one and
the gathered result is bit-identical to the unsharded product (pin P11).

The token all-gather is chunk-pipelined: the local columns are cut into
`chunks` pieces; after a piece is computed on the compute stream its gather is
enqueued on a side stream while the next piece computes.

The compute step is injectable (`compute=`) so the partition / gather logic is
testable on CPU with the gloo backend (tests/test_parallel_gloo.py); on GPUs it
is always the C-ABI SpMM.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

ComputeFn = Callable[[torch.Tensor, torch.Tensor], torch.Tensor]   # (B_cols, out) -> out


def shard_range(n_total: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """Contiguous shard [c0, c1) of n_total columns; shard widths are `align`-multiples
    (16-byte aligned rows for bf16/fp32) except possibly the last."""
    per = -(-n_total // world)
    per = -(-per // align) * align
    c0 = min(n_total, rank * per)
    c1 = min(n_total, (rank + 1) * per)
    return c0, c1


def padded_shard_width(n_total: int, world: int, align: int = 8) -> int:
    per = -(-n_total // world)
    return -(-per // align) * align


def group_range(M: int, g: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of whole groups owned by `rank` under row sharding."""
    G = M // g
    return (rank * G // world) * g, ((rank + 1) * G // world) * g


def aligned_rows(B: torch.Tensor) -> torch.Tensor:
    """B itself when its rows start on 16-byte boundaries (the TMA contract of the C ABI:
    16-byte aligned base and row pitch), else a copy into a buffer whose pitch is rounded up
    to 16 bytes -- a layout copy (device-memory plumbing), no arithmetic."""
    es = B.element_size()
    if B.dim() != 2 or B.shape[1] == 0 or B.device.type != "cuda":
        return B
    if B.stride(1) == 1 and (B.stride(0) * es) % 16 == 0 and B.data_ptr() % 16 == 0:
        return B
    pitch = -(-B.shape[1] * es // 16) * 16 // es
    buf = torch.empty((B.shape[0], pitch), dtype=B.dtype, device=B.device)
    out = buf[:, : B.shape[1]]
    out.copy_(B)
    return out


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def sten_compute(values, idx, n, m, g, plan, out_dtype) -> ComputeFn:
    """The GPU compute step: C_cols = densify(values, idx) @ B_cols through the C ABI."""
    from . import sten

    def fn(B_cols: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        return sten.spmm_grouped_nm(values, idx, B_cols, n, m, g, out=out, plan=plan)
    return fn


class TokenShardedSpmm:
    """C[:, shard] = W_sparse @ B[:, shard] on every rank, optional all-gather of C."""

    def __init__(self, M: int, N_global: int, out_dtype: torch.dtype, device, compute: ComputeFn,
                 chunks: int = 1, group=None):
        self.M, self.N_global = M, N_global
        self.out_dtype, self.device = out_dtype, torch.device(device)
        self.compute = compute
        self.group = group
        self.world, self.rank = _world(group)
        self.n_local = padded_shard_width(N_global, self.world)
        self.chunks = max(1, chunks)
        self.use_streams = self.device.type == "cuda"
        self.comm_stream = torch.cuda.Stream(device=self.device) if self.use_streams else None

    @classmethod
    def from_sten(cls, values, idx, n, m, g, K, N_global, out_dtype=None, chunks=1, group=None):
        from . import sten
        out_dtype = out_dtype or values.dtype
        plan = sten.spmm_plan(n, m, g, values.shape[0], K, N_global, ab_dtype=values.dtype, c_dtype=out_dtype)
        return cls(values.shape[0], N_global, out_dtype, values.device,
                   sten_compute(values, idx, n, m, g, plan, out_dtype), chunks, group)

    def local_range(self) -> tuple[int, int]:
        return shard_range(self.N_global, self.world, self.rank)

    def forward_local(self, B_local: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.M, B_local.shape[1]), dtype=self.out_dtype, device=self.device)
        return self.compute(B_local, out)

    def _chunk_bounds(self):
        step = -(-self.n_local // self.chunks)
        step = -(-step // 8) * 8
        return [(c, min(self.n_local, c + step)) for c in range(0, self.n_local, step)]

    def forward_allgather(self, B_local: torch.Tensor) -> torch.Tensor:
        """Compute the local shard chunk by chunk and all-gather every chunk as soon as it
        is done (side stream on GPUs).  Returns C [M][N_global]."""
        M, nl, world = self.M, self.n_local, self.world
        B_local = aligned_rows(B_local)
        have = B_local.shape[1]
        bounds = self._chunk_bounds()
        staged = []
        compute_stream = torch.cuda.current_stream(self.device) if self.use_streams else None
        for (c0, c1) in bounds:
            piece = torch.zeros((M, c1 - c0), dtype=self.out_dtype, device=self.device)
            hi = min(c1, have)
            if hi > c0:
                self.compute(B_local[:, c0:hi], piece[:, : hi - c0])
            gathered = torch.empty((world * M, c1 - c0), dtype=self.out_dtype, device=self.device)
            if self.use_streams and world > 1:
                ev = torch.cuda.Event()
                ev.record(compute_stream)
                with torch.cuda.stream(self.comm_stream):
                    self.comm_stream.wait_event(ev)
                    dist.all_gather_into_tensor(gathered, piece, group=self.group)
                    piece.record_stream(self.comm_stream)
                    gathered.record_stream(self.comm_stream)
            elif world > 1:
                parts = list(gathered.chunk(world, dim=0))
                dist.all_gather(parts, piece, group=self.group)
            else:
                gathered.copy_(piece)
            staged.append(gathered)
        if self.use_streams and world > 1:
            compute_stream.wait_stream(self.comm_stream)
        # assemble: rank p's local column j is global column p * n_local + j -- one strided copy
        # per chunk ([world][M][cw] gathered block -> columns {p n_local + c0 ..} of every rank p)
        full = torch.empty((M, world, nl), dtype=self.out_dtype, device=self.device)
        for (c0, c1), gathered in zip(bounds, staged):
            full[:, :, c0:c1].copy_(gathered.view(world, M, c1 - c0).permute(1, 0, 2))
        return full.view(M, world * nl)[:, : self.N_global]


class RowShardedSpmm:
    """Rank p owns groups [p*G/P, (p+1)*G/P): C[rows_p, :] = W_p @ B, then all-gather along M."""

    def __init__(self, M_global: int, g: int, N: int, out_dtype: torch.dtype, device, compute: ComputeFn,
                 group=None):
        self.M_global, self.g, self.N = M_global, g, N
        self.out_dtype, self.device = out_dtype, torch.device(device)
        self.compute = compute
        self.group = group
        self.world, self.rank = _world(group)
        self.r0, self.r1 = group_range(M_global, g, self.world, self.rank)

    def forward_allgather(self, B: torch.Tensor) -> torch.Tensor:
        rows = [group_range(self.M_global, self.g, self.world, p) for p in range(self.world)]
        maxr = max(r1 - r0 for r0, r1 in rows)
        local = torch.zeros((maxr, self.N), dtype=self.out_dtype, device=self.device)
        nr = self.r1 - self.r0
        B = aligned_rows(B)
        if nr:
            self.compute(B, local[:nr])
        gathered = torch.empty((self.world * maxr, self.N), dtype=self.out_dtype, device=self.device)
        if self.world > 1:
            if self.device.type == "cuda":
                dist.all_gather_into_tensor(gathered, local, group=self.group)
            else:
                dist.all_gather(list(gathered.chunk(self.world, dim=0)), local, group=self.group)
        else:
            gathered.copy_(local)
        return torch.cat([gathered[p * maxr: p * maxr + (r1 - r0)] for p, (r0, r1) in enumerate(rows)], dim=0)


class FusedAllGatherSpmm:
    """Token sharding with the all-gather fused into the SpMM epilogue over NVLink peer memory.

    The gathered output C [M][N_pad] lives in symmetric memory (one allocation per rank,
    mapped into every peer: ``torch.distributed._symmetric_memory``); each rank's kernel
    (``sten_spmm_grouped_nm_allgather``) stores its C tiles straight into the slot
    [p * n_local, (p + 1) * n_local) of EVERY rank's buffer, so the exchange overlaps the
    math tile by tile and no NCCL call runs; a device-side barrier over the symmetric
    memory handle ends the step.  Needs one GPU per rank with peer access (NVLink /
    NVSwitch); the kernel path itself is tested on one GPU with local stand-in buffers
    (tests/test_gpu_parity.py::test_spmm_fused_allgather_equals_unsharded).
    """

    def __init__(self, values, idx, n, m, g, K, N_global, out_dtype=None, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        from . import sten
        self.values, self.idx, self.n, self.m, self.g = values, idx, n, m, g
        self.M = values.shape[0]
        self.out_dtype = out_dtype or values.dtype
        self.group = group or dist.group.WORLD
        self.world, self.rank = _world(self.group)
        self.N_global = N_global
        self.n_local = padded_shard_width(N_global, self.world)
        # the GLOBAL plan (pin P11), restricted to the fused-epilogue kernel (SIMT).  When the automatic
        # choice for the global shape is another algorithm its tile / split numbers mean something else,
        # so a concrete SIMT plan is used instead (tile 1 exists for fp32 and bf16; one K partition) --
        # identical on every rank and independent of the local width.
        plan = sten.spmm_plan(n, m, g, self.M, K, N_global, ab_dtype=values.dtype, c_dtype=self.out_dtype)
        if plan.algo != sten.ALGO_SIMT:
            plan = sten.make_plan(sten.ALGO_SIMT, split_k=1, tile=1)
        self.plan = plan
        ldc = self.world * self.n_local
        self.buf = symm_mem.empty((self.M, ldc), dtype=self.out_dtype, device=values.device)
        self.handle = symm_mem.rendezvous(self.buf, self.group)
        self.peers = [self.handle.get_buffer(p, (self.M, ldc), self.out_dtype) for p in range(self.world)]

    def forward(self, B_local: torch.Tensor, copy: bool = False) -> torch.Tensor:
        """C [M][N_global] on every rank; B_local = this rank's columns of B.

        The result is a view of the persistent symmetric buffer: it stays valid until the next
        forward() (which overwrites it on every rank); pass copy=True for an independent tensor."""
        from . import sten
        # pre-barrier: no rank may start storing into its peers' buffers while a peer's stream is
        # still reading the previous step's result (write-after-read across ranks)
        B_local = aligned_rows(B_local)
        self.handle.barrier(channel=0)
        sten.spmm_grouped_nm_allgather(self.values, self.idx, B_local, self.n, self.m, self.g, self.peers,
                                       self.rank * self.n_local, plan=self.plan)
        self.handle.barrier(channel=0)          # every peer's stores into this buffer have landed
        out = self.buf[:, : self.N_global]
        return out.clone() if copy else out
