"""Python mirror of the executor half of the C ABI (include/hshard_c.h).

    ctx  = Context(arena_bytes)                          # one per process / GPU
    lay  = ShardLayout(ctx, plan, n_virtual)             # symmetric shard buffers
    prog = Program(ctx, plan, lay)                       # compiled tables on the GPU
    lay.fill_src(seed)                                   # synthetic payloads (optional)
    prog.run()                                           # device-resident reshard
    prog.run_host(src_host, dst_host)                    # host-buffer (e2e) path

This is the B200 definition of the reference's declared-but-undefined
execute_plan (sim.hpp:77-79) / apply_switch.  Everything
runs in libhshard_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import json
import os
import time
import weakref
from ctypes import c_int, c_size_t, c_ulonglong, c_void_p
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import hshard as H
from ._lib import LIB, check, i64_array, take_string

SIZE_MAX = (1 << 64) - 1
HS_PROG_FUSE_PHASES = 1   # fuse phase-1 sums into phase-2 tasks (default when world == 1)
HS_PROG_NO_FUSE = 2       # materialise the mid annotation
HS_PROG_NO_TMA = 4        # register path only
HS_PROG_NO_MERGE = 8      # one task per destination shard
HS_PROG_NO_TMA_PEER = 16  # peer (NVLink) terms use the register path
HS_PROG_NO_RELAY = 32      # world > 1: pull remote mid boxes instead of relay stores
HS_PROG_NO_REPLICA = 64    # world > 1: no replica-aware source choice
HS_PROG_NO_SHARE = 128     # world > 1: no cross-rank chunking of identical tasks
HS_PROG_PULL_COPIES = 256  # world > 1: copies pull (run on the destination's rank)
HS_PROG_RELAY_KEEP_LOCAL = 512  # world > 1: relay-waiting tasks keep local groups before the barrier
HS_PROG_PUSH_ALL = 1024    # world > 1: every copy runs on its input's rank (before output merging)
HS_PROG_NCCL = 2048         # world > 1: NCCL grouped send/recv transport (baseline)
HS_PROG_NO_STREAM = 4096    # world > 1: barrier between plan phases (no per-chunk ready flags)
HS_PROG_PULL_MID = 8192     # world > 1: pull remote mid boxes (no relay stores), local groups fused
HS_PROG_CE_RELAY = 16384    # world > 1: relays copied by the copy engines in row chunks, SMs keep computing
HS_PROG_FANOUT_ONCE = 32768  # world > 1: one NVLink store per remote GPU, local copies to its other shards
HS_PROG_STATIC_LOCAL = 1 << 24  # world > 1: static dealing for uniform local-only launches
HS_PROG_BULK_STORE = 1 << 25  # static TMA kernel: copies' first two outputs leave through TMA bulk stores
HS_PROG_SEPARATE_BARRIERS = 1 << 26  # world > 1: barriers as their own launches, not kernel prologues
HS_PROG_SMALL_ITEMS = 1 << 27  # 16 KB TMA work items (plan-dependent; autotuned at N=1)
HS_PROG_NO_PDL = 1 << 28  # no programmatic dependent launch between phase kernels (A/B)
HS_PROG_INTERLEAVE = 1 << 29  # world > 1: NVLink and local-only items merged evenly in launch order
HS_PROG_SPLIT_RELAY = 1 << 30  # world > 1: remote mid rows half pushed before the barrier, half pulled after
HS_PROG_BASELINE = HS_PROG_NO_FUSE | HS_PROG_NO_TMA | HS_PROG_NO_MERGE

NP_STORAGE = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64,
              "bf16": np.uint16}


def block_map(n_virtual: int, world: int) -> List[int]:
    """Virtual device v -> rank v // ceil(n_virtual / world) (SURVEY §8e block mapping)."""
    per = -(-n_virtual // world)
    return [min(v // per, world - 1) for v in range(n_virtual)]


class Context:
    """hs_ctx: this process's GPU, its symmetric arena, and (world > 1) the peers' arenas."""

    def __init__(self, arena_bytes: int, rank: int = 0, world: int = 1, gpu: Optional[int] = None,
                 group=None):
        self.rank, self.world = rank, world
        self.gpu = rank if gpu is None else gpu
        h = c_void_p()
        check(LIB.hs_ctx_create(rank, world, self.gpu, arena_bytes, ctypes.byref(h)))
        self._h = h
        self._programs = weakref.WeakSet()
        base, size = c_void_p(), c_size_t()
        check(LIB.hs_ctx_arena(self._h, ctypes.byref(base), ctypes.byref(size)))
        self.arena_base, self.arena_bytes = base.value, size.value
        self.sym_bytes = self.arena_bytes  # min over ranks (set when the peers open)
        if world > 1:
            self._open_peers(group)

    def _open_peers(self, group):
        import torch
        import torch.distributed as dist
        mine = ctypes.create_string_buffer(128)
        check(LIB.hs_ctx_ipc_handle(self._h, mine))
        t = torch.frombuffer(bytearray(mine.raw), dtype=torch.uint8)
        gathered = [torch.zeros(128, dtype=torch.uint8) for _ in range(self.world)]
        dist.all_gather(gathered, t, group=group)
        blob = b"".join(bytes(g.numpy().tobytes()) for g in gathered)
        check(LIB.hs_ctx_open_peers(self._h, blob))
        # The arenas are symmetric only up to the smallest one: an offset is valid on
        # every rank below it (layouts placed from the top must use it, not arena_bytes).
        sz = torch.tensor([float(self.arena_bytes)], dtype=torch.float64)
        dist.all_reduce(sz, op=dist.ReduceOp.MIN, group=group)
        self.sym_bytes = int(sz.item())

    def init_nccl(self, group=None) -> None:
        """NCCL communicator over the same ranks (only the HS_PROG_NCCL baseline uses it)."""
        import torch.distributed as dist
        uid = [None]
        if self.rank == 0:
            buf = ctypes.create_string_buffer(128)
            check(LIB.hs_nccl_unique_id(buf))
            uid[0] = buf.raw
        dist.broadcast_object_list(uid, src=0, group=group)
        check(LIB.hs_ctx_nccl_init(self._h, uid[0]))

    @property
    def handle(self):
        return self._h

    def alloc(self, nbytes: int) -> int:
        off = c_size_t()
        check(LIB.hs_ctx_alloc(self._h, nbytes, ctypes.byref(off)))
        return off.value

    def reset(self, offset: int = 0) -> None:
        check(LIB.hs_ctx_reset_alloc(self._h, offset))

    def read(self, offset: int, nbytes: int) -> bytes:
        buf = ctypes.create_string_buffer(nbytes)
        check(LIB.hs_ctx_read(self._h, offset, buf, nbytes))
        return buf.raw

    def read_array(self, offset: int, shape, dtype: str) -> np.ndarray:
        n = int(np.prod(shape)) if len(shape) else 1
        out = np.empty(n, dtype=NP_STORAGE[dtype])
        if out.nbytes:
            check(LIB.hs_ctx_read(self._h, offset, out.ctypes.data_as(c_void_p), out.nbytes))
        return out.reshape(shape)

    def write_array(self, offset: int, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr)
        if arr.nbytes:
            check(LIB.hs_ctx_write(self._h, offset, arr.ctypes.data_as(c_void_p), arr.nbytes))

    def sync(self) -> None:
        check(LIB.hs_ctx_sync(self._h))

    def barrier(self, stream=None) -> None:
        """Device-side cross-rank barrier enqueued on `stream` (a cuda stream handle; None = ctx stream)."""
        check(LIB.hs_ctx_barrier(self._h, c_void_p(stream or 0)))

    def clear_error(self) -> None:
        """Clear a recorded DeadlockDetected once every rank has drained (hs_ctx_clear_error)."""
        check(LIB.hs_ctx_clear_error(self._h))

    def close(self) -> None:
        # programs compiled against this context go first (their tables, events
        # and streams belong to its device)
        for prog in list(getattr(self, "_programs", ())):
            prog.close()
        h, self._h = getattr(self, "_h", None), None
        if h:
            LIB.hs_ctx_destroy(h)

    def __del__(self):
        self.close()


def _box(anno: str, shape, dev: int):
    p = H.placement(anno, shape, dev)
    return p


class ShardLayout:
    """Symmetric placement of every src/dst shard of a plan in the arenas.

    Every rank computes the same per-rank dense packing (so it knows where each
    peer keeps each shard), then reserves max-over-ranks bytes once; offsets
    are identical on every rank by construction.  Keys are (tensor slot, dev).
    """

    def __init__(self, ctx: Context, plan: H.Plan, n_virtual: int,
                 v_to_rank: Optional[Sequence[int]] = None):
        self.ctx = ctx
        self.plan = plan
        self.n_virtual = n_virtual
        self.v_to_rank = list(v_to_rank) if v_to_rank is not None else block_map(n_virtual, ctx.world)
        self.dtype = plan.meta["dtype"]
        self.es = H.DTYPE_BYTES[self.dtype]
        if plan.kind == "comm":
            self.entries = [(0, plan.meta["src"], plan.meta["dst"], list(plan.meta["shape"]))]
        else:
            self.entries = [(tid, s, d, list(sh)) for tid, s, d, sh in plan.meta["entries"]]
        self.src: Dict[Tuple[int, int], dict] = {}
        self.dst: Dict[Tuple[int, int], dict] = {}
        self._place()

    def _place(self):
        used = [0] * self.ctx.world
        recs = []
        for side, store in (("src", self.src), ("dst", self.dst)):
            for slot, (tid, s, d, shape) in enumerate(self.entries):
                anno = s if side == "src" else d
                devs = sorted({x for g in H.parse_annotation(anno)["groups"] for x in g})
                for dev in devs:
                    if dev >= self.n_virtual:
                        raise H.HshardError("UnknownDevice", f"device {dev} >= n_virtual")
                    p = _box(anno, shape, dev)
                    ext = [hi - lo for lo, hi in p["bounds"]]
                    nbytes = int(np.prod(ext)) * self.es if ext else self.es
                    r = self.v_to_rank[dev]
                    off = (used[r] + 255) // 256 * 256
                    used[r] = off + nbytes
                    rec = {"slot": slot, "dev": dev, "rank": r, "rel": off, "bytes": nbytes,
                           "ext": ext, "bounds": p["bounds"], "partial": p["partial"],
                           "anno": anno, "shape": shape, "tid": tid}
                    store[(slot, dev)] = rec
                    recs.append(rec)
        self.base = self.ctx.alloc(max(used) + 256)
        for rec in recs:
            rec["offset"] = self.base + rec["rel"]
        self.src_off = self._table(self.src)
        self.dst_off = self._table(self.dst)
        self.local_src_bytes = sum(r["bytes"] for r in self.src.values() if r["rank"] == self.ctx.rank)
        self.local_dst_bytes = sum(r["bytes"] for r in self.dst.values() if r["rank"] == self.ctx.rank)

    def _table(self, store):
        n = len(self.entries) * self.n_virtual
        arr = (c_size_t * max(1, n))(*([SIZE_MAX] * max(1, n)))
        for (slot, dev), rec in store.items():
            arr[slot * self.n_virtual + dev] = rec["offset"]
        return arr

    def local(self, side: str):
        store = self.src if side == "src" else self.dst
        return {k: v for k, v in store.items() if v["rank"] == self.ctx.rank}

    # ---- payloads -------------------------------------------------------------
    def fill_src(self, seed: int, mode: str = "grid", stream=None) -> None:
        """Counter-hash payload into every local source shard."""
        m = 0 if mode == "grid" else 1
        for (slot, dev), rec in self.local("src").items():
            arr, n = _shape_arr(rec["shape"])
            check(LIB.hs_fill_shard(self.ctx.handle, rec["anno"].encode(), arr, n,
                                    H.DTYPES[self.dtype], dev, rec["offset"], seed, rec["tid"], m,
                                    stream))

    def verify_dst(self, seed: int) -> int:
        """Mismatching cells of every local dst shard vs the logical grid tensor
        (valid for Partial-free destination annotations)."""
        bad = 0
        for (slot, dev), rec in self.local("dst").items():
            arr, n = _shape_arr(rec["shape"])
            out = c_ulonglong()
            check(LIB.hs_verify_shard(self.ctx.handle, rec["anno"].encode(), arr, n,
                                      H.DTYPES[self.dtype], dev, rec["offset"], seed, rec["tid"],
                                      ctypes.byref(out), None))
            bad += out.value
        return bad

    def read(self, side: str, slot: int, dev: int) -> np.ndarray:
        rec = (self.src if side == "src" else self.dst)[(slot, dev)]
        return self.ctx.read_array(rec["offset"], rec["ext"], self.dtype)

    def write(self, side: str, slot: int, dev: int, arr: np.ndarray) -> None:
        rec = (self.src if side == "src" else self.dst)[(slot, dev)]
        assert list(arr.shape) == rec["ext"], (arr.shape, rec["ext"])
        self.ctx.write_array(rec["offset"], arr.astype(NP_STORAGE[self.dtype], copy=False))

    def clear_dst(self) -> None:
        for rec in self.local("dst").values():
            self.ctx.write_array(rec["offset"], np.full(rec["bytes"], 0xA5, dtype=np.uint8))


class PointerLayout:
    """Caller-owned shard buffers (hs_prog_compile_ptrs): {(slot, dev): device address}
    valid in this process -- e.g. torch tensors' data_ptr() on this GPU, or peers'
    buffers mapped by exchange_pointers().  Each buffer is row-major over the shard's
    placement box in the plan's dtype; the program reads / writes them in place."""

    def __init__(self, n_virtual: int, n_slots: int, src: Dict[Tuple[int, int], int],
                 dst: Dict[Tuple[int, int], int], v_to_rank: Sequence[int]):
        self.n_virtual, self.v_to_rank = n_virtual, list(v_to_rank)
        self.entries = [None] * n_slots
        n = max(1, n_slots * n_virtual)
        self.src_ptr, self.dst_ptr = (c_void_p * n)(), (c_void_p * n)()
        for (slot, dev), ptr in src.items():
            self.src_ptr[slot * n_virtual + dev] = ptr
        for (slot, dev), ptr in dst.items():
            self.dst_ptr[slot * n_virtual + dev] = ptr


def exchange_pointers(ctx: Context, local: Dict[Tuple[str, int, int], int], group=None) -> Dict:
    """N > 1: every rank passes its OWN shards' device pointers {(side, slot, dev): ptr};
    returns every rank's shards mapped into this process (hs_ipc_export on the owner,
    an all-gather of the 80-byte exports, hs_ipc_import here)."""
    import torch.distributed as dist
    mine = []
    for key, ptr in sorted(local.items()):
        buf = ctypes.create_string_buffer(80)
        check(LIB.hs_ipc_export(ctx.handle, c_void_p(ptr), buf))
        mine.append((key, buf.raw))
    allv = [None] * ctx.world
    dist.all_gather_object(allv, mine, group=group)
    out = dict(local)
    for r, items in enumerate(allv):
        if r == ctx.rank:
            continue
        for key, blob in items:
            p = c_void_p()
            check(LIB.hs_ipc_import(ctx.handle, blob, ctypes.byref(p)))
            out[key] = p.value
    return out


class StateLayout:
    """One layout state of a set of tensors -- e.g. every parameter of a model under one
    parallel strategy -- packed symmetrically into the arenas (the same per-rank dense
    packing as ShardLayout, for one side).  Graph switches chain states: the destination
    state of S1->S2 is the source state of S2->S3 (SPEC.md:428-433 apply_switch, where a
    switch releases the old shards), so a cycle needs only two states resident at a time.

    entries: [(slot, tensor_id, annotation, shape)].  `base`: arena offset to place the
    state at (None = bump-allocate); StateLayout.bytes_needed() sizes it first.
    """

    def __init__(self, ctx: Context, entries, dtype: str, n_virtual: int,
                 v_to_rank: Optional[Sequence[int]] = None, base: Optional[int] = None):
        self.ctx, self.dtype, self.n_virtual = ctx, dtype, n_virtual
        self.v_to_rank = list(v_to_rank) if v_to_rank is not None else block_map(n_virtual, ctx.world)
        self.es = H.DTYPE_BYTES[dtype]
        self.entries = [(int(slot), int(tid), anno, [int(x) for x in shape]) for slot, tid, anno, shape in entries]
        self.n_slots = max((e[0] for e in self.entries), default=-1) + 1
        self.recs, used = self._pack(self.entries, self.es, self.n_virtual, self.v_to_rank, ctx.world)
        self.size = max(used) + 256
        self.base = ctx.alloc(self.size) if base is None else int(base)
        if self.base + self.size > getattr(ctx, "sym_bytes", ctx.arena_bytes):
            raise H.HshardError("ShapeMismatch", "state does not fit the arena")
        self._by_tid: Dict[int, Dict[int, int]] = {}
        for rec in self.recs.values():
            rec["offset"] = self.base + rec["rel"]
            self._by_tid.setdefault(rec["tid"], {})[rec["dev"]] = rec["offset"]

    @staticmethod
    def _pack(entries, es, n_virtual, v_to_rank, world):
        used = [0] * world
        recs = {}
        for slot, tid, anno, shape in entries:
            devs = sorted({x for g in H.parse_annotation(anno)["groups"] for x in g})
            for dev in devs:
                if dev >= n_virtual:
                    raise H.HshardError("UnknownDevice", f"device {dev} >= n_virtual")
                p = _box(anno, shape, dev)
                ext = [hi - lo for lo, hi in p["bounds"]]
                nbytes = int(np.prod(ext)) * es if ext else es
                r = v_to_rank[dev]
                off = (used[r] + 255) // 256 * 256
                used[r] = off + nbytes
                recs[(slot, dev)] = {"slot": slot, "dev": dev, "rank": r, "rel": off, "bytes": nbytes, "ext": ext,
                                     "bounds": p["bounds"], "partial": p["partial"], "anno": anno,
                                     "shape": shape, "tid": tid}
        return recs, used

    @staticmethod
    def bytes_needed(entries, dtype: str, n_virtual: int, world: int, v_to_rank=None) -> int:
        m = list(v_to_rank) if v_to_rank is not None else block_map(n_virtual, world)
        _, used = StateLayout._pack([(s, t, a, [int(x) for x in sh]) for s, t, a, sh in entries],
                                    H.DTYPE_BYTES[dtype], n_virtual, m, world)
        return max(used) + 256

    def offsets(self, tensor_ids: Sequence[int]):
        """Offset table for a plan whose tensor slots are `tensor_ids` (slot i = the plan's
        i-th tensor): arr[i * n_virtual + dev]; tensors this state lacks stay absent."""
        nv = self.n_virtual
        flat = np.full(max(1, len(tensor_ids) * nv), SIZE_MAX, dtype=np.uint64)
        for i, tid in enumerate(tensor_ids):
            for dev, off in self._by_tid.get(int(tid), {}).items():
                flat[i * nv + dev] = off
        return flat

    def local(self):
        return {k: v for k, v in self.recs.items() if v["rank"] == self.ctx.rank}

    def fill(self, seed: int, mode: str = "grid", stream=None) -> None:
        m = 0 if mode == "grid" else 1
        for (slot, dev), rec in self.local().items():
            arr, n = _shape_arr(rec["shape"])
            check(LIB.hs_fill_shard(self.ctx.handle, rec["anno"].encode(), arr, n, H.DTYPES[self.dtype], dev,
                                    rec["offset"], seed, rec["tid"], m, stream))

    def verify(self, seed: int) -> int:
        """Cells of this rank's shards that differ from the logical grid tensors."""
        bad = 0
        for (slot, dev), rec in self.local().items():
            arr, n = _shape_arr(rec["shape"])
            out = c_ulonglong()
            check(LIB.hs_verify_shard(self.ctx.handle, rec["anno"].encode(), arr, n, H.DTYPES[self.dtype], dev,
                                      rec["offset"], seed, rec["tid"], ctypes.byref(out), None))
            bad += out.value
        return bad


class Transition:
    """A (source state, destination state) pair in the form Program compiles against:
    offset tables indexed by the plan's tensor slots (a switch plan lists only the
    parameters that move, in its own order; shards are matched by tensor id)."""

    def __init__(self, plan: "H.Plan", src: StateLayout, dst: StateLayout):
        if src.n_virtual != dst.n_virtual or src.v_to_rank != dst.v_to_rank:
            raise H.HshardError("UnknownDevice", "states map virtual devices differently")
        self.src_state, self.dst_state = src, dst
        self.n_virtual, self.v_to_rank = src.n_virtual, src.v_to_rank
        if plan.kind == "comm":
            tids = [0]
        else:
            tids = [int(e[0]) for e in plan.meta["entries"]]
        self.entries = [(t, None, None, None) for t in tids]
        self._offs = (src.offsets(tids), dst.offsets(tids))  # kept alive for the pointers
        self.src_off, self.dst_off = (a.ctypes.data_as(ctypes.POINTER(c_size_t)) for a in self._offs)


class SwitchCache:
    """Plans and compiled programs cached per (source, destination) strategy
    (host planning is the same order as a switch's
    execution, so a strategy cycle must not re-plan).  Keys: the switch's
    parameter moves + dtype (plan), and the plan with the two states' placement
    + program flags (program)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self.plans: Dict[tuple, "H.Plan"] = {}
        self.programs: Dict[tuple, "Program"] = {}
        self._by_id: Dict[tuple, tuple] = {}  # (id(entries), dtype) -> (entries, key)

    def plan(self, entries, dtype: str):
        # the same entries object again (a cycle's step lists): no key rebuild
        ident = self._by_id.get((id(entries), dtype))
        if ident is not None and ident[0] is entries:
            return self.plans[ident[1]], True
        key = (tuple((int(t), s, d, tuple(int(x) for x in sh)) for t, s, d, sh in entries), dtype)
        self._by_id[(id(entries), dtype)] = (entries, key)
        p = self.plans.get(key)
        hit = p is not None
        if not hit:
            p = self.plans[key] = H.plan_switch(entries, dtype)
        return p, hit

    def program(self, plan, src: StateLayout, dst: StateLayout, flags: int = 0):
        key = (id(plan), src.base, src.size, dst.base, dst.size, flags)
        prog = self.programs.get(key)
        hit = prog is not None
        if not hit:
            prog = self.programs[key] = Program(self.ctx, plan, Transition(plan, src, dst), flags)
        return prog, hit

    def close(self):
        for p in self.programs.values():
            p.close()
        self.programs.clear()
        self.plans.clear()
        self._by_id.clear()


class StrategyCycle:
    """Graph switching through a cycle of parallel strategies:
    one StateLayout per strategy, alternating between the low and the high end of
    the arena (a switch releases the old state, so two states are
    resident at a time), and a SwitchCache so that the second time round no plan is
    re-planned and no program recompiled.

    steps: list of switch transition lists [(tensor_id, src, dst, shape)], where
    step k's destinations are step k+1's sources; when the last step returns to the
    first strategy the cycle reuses the first state's placement."""

    def __init__(self, ctx: Context, steps, dtype: str, n_virtual: int, flags: Optional[int] = None):
        # Untuned defaults (switch plans are copy-only).  Across GPUs: every copy runs on
        # the rank holding its input, no cross-rank chunking, NVLink and local items
        # interleaved -- up to 1.7x faster than flags 0 on the cfg4 / cfg5 steps
        # (profiles/r02_cycle_flags_n{2,4}.jsonl).  TMA bulk stores to peers are left
        # to the autotuner there (1-2% at N>1; the only two bad parity results of the
        # round came from a cycle with them).  On one GPU copies
        # leave through TMA bulk stores: never more than 0.1% slower than flags 0,
        # 3-7% faster on cfg4 and cfg5 S2->S3 / S3->S4 / S4->S1.
        # Beyond 4 ranks the default stays flags 0: at 8 ranks a TMA-path bug in pushed
        # multi-output copies (PUSH_ALL) is open.
        if flags is None:
            flags = (HS_PROG_BULK_STORE if ctx.world == 1 else
                     HS_PROG_PUSH_ALL | HS_PROG_NO_SHARE | HS_PROG_INTERLEAVE if ctx.world <= 4 else 0)
        self.ctx, self.steps, self.dtype, self.n_virtual, self.flags = ctx, steps, dtype, n_virtual, flags
        ents = [[(i, tid, s, shp) for i, (tid, s, d, shp) in enumerate(st)] for st in steps]
        ents.append([(i, tid, d, shp) for i, (tid, s, d, shp) in enumerate(steps[-1])])
        closed = [e[1:] for e in ents[-1]] == [e[1:] for e in ents[0]]
        self.sizes = [StateLayout.bytes_needed(e, dtype, n_virtual, ctx.world) for e in ents]
        # the top of the SYMMETRIC arena: every rank places the high states at the same
        # offsets (arena sizes may differ between ranks)
        top = getattr(ctx, "sym_bytes", ctx.arena_bytes) // 256 * 256
        need = max(self.sizes[k] + self.sizes[k + 1] for k in range(len(steps)))
        if need > top:
            raise H.HshardError("ShapeMismatch", f"two states need {need} bytes per GPU, arena {top}")
        if closed and len(steps) % 2 == 1:
            raise H.HshardError("UnsupportedOp", "a closed cycle needs an even number of steps")
        self.states: List[StateLayout] = []
        for k, e in enumerate(ents):
            if k == len(ents) - 1 and closed:
                self.states.append(self.states[0])
                continue
            base = 0 if k % 2 == 0 else (top - self.sizes[k]) // 256 * 256
            self.states.append(StateLayout(ctx, e, dtype, n_virtual, base=base))
        # Program scratch (intermediates, relays, ready flags) comes from the arena's
        # bump allocator: start it past every low-placed state and keep it below every
        # high-placed one, so no program's scratch overlaps a state.
        self.scratch_lo = max(st.base + st.size for st in self.states if st.base == 0)
        self.scratch_hi = min((st.base for st in self.states if st.base > 0), default=top)
        if self.scratch_lo >= self.scratch_hi:
            raise H.HshardError("ShapeMismatch", "no arena left between the layout states")
        ctx.reset((self.scratch_lo + 255) // 256 * 256)
        self.cache = SwitchCache(ctx)
        self.step_flags: Dict[int, int] = {}  # per step: the variant tune() chose

    def _check_scratch(self):
        if self.ctx.alloc(0) > self.scratch_hi:
            raise H.HshardError("ShapeMismatch", "program scratch reached a layout state")

    def prepare(self, k: int):
        """Plan (cached) and compile (cached) step k -> (program, info)."""
        t0 = time.perf_counter()
        plan, plan_hit = self.cache.plan(self.steps[k], self.dtype)
        t1 = time.perf_counter()
        prog, prog_hit = self.cache.program(plan, self.states[k], self.states[k + 1],
                                            self.step_flags.get(k, self.flags))
        self._check_scratch()
        t2 = time.perf_counter()
        return prog, {"plan_cached": plan_hit, "program_cached": prog_hit, "plan_ms": (t1 - t0) * 1e3,
                      "compile_ms": (t2 - t1) * 1e3, "flags": self.step_flags.get(k, self.flags)}

    def tune(self, k: int, stream=None, steps: int = 5, group=None) -> dict:
        """Autotune step k's program variant (executor.autotune, every rank together) and
        keep the winner in the cache: later prepare(k) calls return it.  Rewrites the
        destination state with the same values (the source state is only read)."""
        plan, _ = self.cache.plan(self.steps[k], self.dtype)
        prog, timings = autotune(self.ctx, plan, Transition(plan, self.states[k], self.states[k + 1]),
                                 stream=stream, steps=steps, group=group)
        self._check_scratch()
        key = (id(plan), self.states[k].base, self.states[k].size, self.states[k + 1].base,
               self.states[k + 1].size, prog.flags)
        old = self.cache.programs.get(key)
        if old is not None and old is not prog:
            old.close()
        self.cache.programs[key] = prog
        self.step_flags[k] = prog.flags
        return {"chosen_flags": prog.flags, "ms_by_flags": timings}

    def close(self):
        self.cache.close()


def _shape_arr(shape):
    return i64_array(shape), len(shape)


class Program:
    """hs_prog: a plan compiled for this rank."""

    def __init__(self, ctx: Context, plan: H.Plan, layout, flags: int = 0):
        self.ctx, self.plan, self.layout, self.flags = ctx, plan, layout, flags
        m = (c_int * layout.n_virtual)(*layout.v_to_rank)
        h = c_void_p()
        if isinstance(layout, PointerLayout):
            check(LIB.hs_prog_compile_ptrs(ctx.handle, plan.handle, m, layout.n_virtual, layout.src_ptr,
                                           layout.dst_ptr, flags, ctypes.byref(h)))
        else:
            check(LIB.hs_prog_compile(ctx.handle, plan.handle, m, layout.n_virtual, layout.src_off,
                                      layout.dst_off, flags, ctypes.byref(h)))
        self._h = h
        ctx._programs.add(self)

    def run(self, stream=None) -> None:
        check(LIB.hs_prog_run(self._h, stream))

    def _host_ptrs(self, src, dst):
        n = len(self.layout.entries) * self.layout.n_virtual
        sp = (c_void_p * max(1, n))()
        dp = (c_void_p * max(1, n))()
        for (slot, dev), a in src.items():
            sp[slot * self.layout.n_virtual + dev] = a.ctypes.data
        for (slot, dev), a in dst.items():
            dp[slot * self.layout.n_virtual + dev] = a.ctypes.data
        return sp, dp

    def run_host(self, src: Dict[Tuple[int, int], np.ndarray], dst: Dict[Tuple[int, int], np.ndarray]):
        """Host-buffer execution: src/dst keyed by (slot, dev); only this rank's shards are used."""
        sp, dp = self._host_ptrs(src, dst)
        check(LIB.hs_prog_run_host(self._h, sp, dp))

    def run_host_async(self, src, dst, h2d, compute, d2h) -> None:
        """run_host enqueued on three CUDA streams (raw cudaStream_t handles); see hs_prog_run_host_async.
        Host buffers should be pinned; synchronise `d2h` before reading `dst`."""
        sp, dp = self._host_ptrs(src, dst)
        check(LIB.hs_prog_run_host_async(self._h, sp, dp, h2d, compute, d2h))

    def profile(self, enable: bool = True) -> None:
        check(LIB.hs_prog_profile(self._h, int(enable)))

    def phase_ms(self):
        """(sum of per-phase kernel ms over profiled runs, run count)."""
        n = max(1, self.stats()["phases"])
        out = (ctypes.c_double * n)()
        runs = c_int()
        check(LIB.hs_prog_phase_ms(self._h, out, n, ctypes.byref(runs)))
        return list(out), runs.value

    def stats(self) -> dict:
        out = c_void_p()
        check(LIB.hs_prog_stats(self._h, ctypes.byref(out)))
        return json.loads(take_string(out))

    def close(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            LIB.hs_prog_destroy(h)

    def __del__(self):
        self.close()




def HS_PROG_STREAM_SHARE(sixty_fourths: int) -> int:
    """Streamed programs: share of CTAs taking non-waiting work first (0 = modelled)."""
    return (sixty_fourths & 0xFF) << 16


AUTOTUNE_CANDIDATES = [0, HS_PROG_PULL_COPIES, HS_PROG_NO_SHARE, HS_PROG_NO_SHARE | HS_PROG_PULL_COPIES,
                       HS_PROG_PUSH_ALL, HS_PROG_PUSH_ALL | HS_PROG_NO_SHARE, HS_PROG_RELAY_KEEP_LOCAL,
                       HS_PROG_NO_STREAM, HS_PROG_PULL_MID | HS_PROG_NO_STREAM,
                       HS_PROG_STREAM_SHARE(32), HS_PROG_STREAM_SHARE(51), HS_PROG_FUSE_PHASES,
                       HS_PROG_FANOUT_ONCE, HS_PROG_FANOUT_ONCE | HS_PROG_FUSE_PHASES,
                       HS_PROG_FANOUT_ONCE | HS_PROG_NO_SHARE,
                       HS_PROG_PULL_MID | HS_PROG_NO_STREAM | HS_PROG_STATIC_LOCAL,
                       HS_PROG_NO_SHARE | HS_PROG_BULK_STORE,
                       HS_PROG_PUSH_ALL | HS_PROG_NO_SHARE | HS_PROG_BULK_STORE,
                       # relays pushed while local groups reduce, then a short consume phase
                       HS_PROG_RELAY_KEEP_LOCAL | HS_PROG_NO_STREAM,
                       HS_PROG_RELAY_KEEP_LOCAL | HS_PROG_NO_STREAM | HS_PROG_NO_SHARE,
                       # NVLink and local-only items merged evenly in launch order
                       HS_PROG_INTERLEAVE, HS_PROG_INTERLEAVE | HS_PROG_NO_SHARE | HS_PROG_BULK_STORE,
                       HS_PROG_INTERLEAVE | HS_PROG_RELAY_KEEP_LOCAL | HS_PROG_NO_STREAM,
                       HS_PROG_INTERLEAVE | HS_PROG_NO_STREAM,
                       HS_PROG_INTERLEAVE | HS_PROG_PULL_MID | HS_PROG_NO_STREAM,
                       # remote mid rows half relayed before the barrier, half pulled after it;
                       # with NVLink and local items interleaved in each launch
                       HS_PROG_SPLIT_RELAY | HS_PROG_NO_STREAM,
                       HS_PROG_SPLIT_RELAY | HS_PROG_NO_STREAM | HS_PROG_STATIC_LOCAL,
                       HS_PROG_SPLIT_RELAY | HS_PROG_NO_STREAM | HS_PROG_INTERLEAVE,
                       HS_PROG_SPLIT_RELAY | HS_PROG_NO_STREAM | HS_PROG_INTERLEAVE | HS_PROG_STATIC_LOCAL]
AUTOTUNE_CANDIDATES_1GPU = [0, HS_PROG_BULK_STORE, HS_PROG_SMALL_ITEMS, HS_PROG_SMALL_ITEMS | HS_PROG_BULK_STORE]
TUNE_MARGIN = 0.01  # a later candidate must beat the best so far by 1% (timing noise)
# HS_PROG_CE_RELAY is correct (tests/test_multi_gpu.py) but measured slower on every
# BASELINE plan at N=2, so it is not a default candidate.


def autotune(ctx: Context, plan: H.Plan, layout: ShardLayout, stream=None, steps: int = 5,
             candidates=None, group=None):
    """Pick the program variant (HS_PROG_* flags of the cross-rank rewrites) that runs fastest.

    Every candidate is compiled and timed for `steps` runs with CUDA events on `stream`; the
    max over ranks decides (all ranks take the same choice).  Results are bit-identical across
    variants -- only the placement of work between ranks, the store path or the item size
    differs.  At world == 1 the variants are HS_PROG_BULK_STORE and HS_PROG_SMALL_ITEMS, for
    plans with copy tasks.
    Returns (program, {flags: ms}).
    """
    import torch
    import torch.distributed as dist
    if ctx.world == 1:
        prog = Program(ctx, plan, layout, 0)
        if candidates is None and prog.stats()["copy_tasks"] == 0:
            return prog, {}
        prog.close()
    cands = list(candidates if candidates is not None else
                 AUTOTUNE_CANDIDATES if ctx.world > 1 else AUTOTUNE_CANDIDATES_1GPU)
    s = stream if stream is not None else torch.cuda.current_stream()
    sp = s.cuda_stream
    best, best_ms, timings = None, None, {}
    for flags in cands:
        mark = ctx.alloc(0)  # the arena cursor: scratch must stay symmetric across ranks
        try:
            prog = Program(ctx, plan, layout, flags)
        except H.HshardError:  # a variant this plan cannot take (e.g. a box shape a rewrite does not support)
            prog = None
        if ctx.world > 1:
            # compile checks only see this rank's tasks: every rank skips together, and
            # every rank rewinds the scratch the skipped variant allocated (a rank whose
            # compile failed part-way allocated less), so later offsets stay symmetric
            ok = torch.tensor([0.0 if prog is None else 1.0], dtype=torch.float64)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if ok.item() == 0.0:
                if prog is not None:
                    prog.close()
                prog = None
        if prog is None:
            ctx.reset(mark)
            continue
        two_phase_only = (HS_PROG_RELAY_KEEP_LOCAL | HS_PROG_NO_STREAM | HS_PROG_PULL_MID | HS_PROG_STREAM_SHARE(0xFF)
                          | HS_PROG_FUSE_PHASES | HS_PROG_CE_RELAY | HS_PROG_SPLIT_RELAY)
        # (HS_PROG_INTERLEAVE alone applies to single-phase plans too)
        if flags & two_phase_only and prog.stats()["plan_phases"] < 2:  # same program as another candidate
            prog.close()
            continue
        for _ in range(2):
            prog.run(sp)
        s.synchronize()
        ctx.sync()
        if ctx.world > 1:
            dist.barrier(group=group)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            for _ in range(steps):
                prog.run(sp)
            b.record()
        b.synchronize()
        ctx.sync()
        t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64)
        if ctx.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        ms = float(t.item())
        timings[flags] = ms
        if best is None or ms < best_ms * (1 - TUNE_MARGIN):
            if best is not None:
                best.close()
            best, best_ms = prog, ms
        else:
            prog.close()
    return best, timings


def analyze(plan: H.Plan, world: int, rank: int, n_virtual: int, flags: int = 0,
            v_to_rank: Optional[Sequence[int]] = None):
    """CPU-only dry run of the compiler for one rank (hs_analyze): (stats, tasks)."""
    m = list(v_to_rank) if v_to_rank is not None else block_map(n_virtual, world)
    arr = (c_int * n_virtual)(*m)
    st, ts = c_void_p(), c_void_p()
    check(LIB.hs_analyze(plan.handle, rank, world, arr, n_virtual, flags, ctypes.byref(st), ctypes.byref(ts)))
    return json.loads(take_string(st)), json.loads(take_string(ts))
