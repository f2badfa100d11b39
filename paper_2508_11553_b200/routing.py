"""Multi-GPU session sharding and cross-shard query routing on one node.

Sessions are independent (the reference keeps one trie + lock per session,
trajectory.py:101-104, 137-145), so the store is sharded by session across GPUs, one
process per GPU: ``owner(gsid) = splitmix64(gsid) mod nranks``.

Host-originated requests (every reference entry point) are sent by the host straight to
the owner's store — no collective.  GPU-originated batches (config 5: each rank holds a
batch of queries in HBM for sessions owned anywhere) use ``Router.match``:

1. ``tm_route_prepare`` buckets the local batch by owner inside this rank's IPC-shared
   region and packs the tokens of the queries other ranks own into 18-bit planes;
2. a cross-rank barrier;
3. every owner's K1 kernel reads its queries directly from the requesters' regions over
   NVLink (P2P loads) and writes matched / parent / dup back into them (P2P stores) —
   the exchange is fused into the match kernel;
4. a second barrier publishes the results to the requesters.

By default (``sync="device"``, ``tm_match_routed_sync``) both barriers are epoch flags
in the region headers written and polled by the kernels themselves over NVLink — no
collective library call per batch.  ``sync="nccl"`` (``tm_match_routed``) brackets the
kernel with one-element NCCL all-reduces instead.  ``match_pipelined`` runs a stream of
batches over two regions: batch k+1 is bucketed and packed on a side stream while batch k
is exchanged and matched.  Measured alternatives kept behind flags:
``Router(push=True)`` has requesters write the planes into the owners' inboxes instead of
owners pulling them, and ``match_pipelined(defer_done=True)`` waits for the owners' done
flags on a stream of its own.  PyTorch provides the process group
(setup plumbing: the IPC handle exchange); routing and matching run in the CUDA kernels
behind include/tmstore.h.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check
from .store import DeviceStore

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def owner_of(gsid, nranks: int) -> np.ndarray:
    """Owner rank of global session ids (same function as the device's owner_of)."""
    g = np.asarray(gsid, dtype=np.int64).astype(np.uint64)
    with np.errstate(over="ignore"):
        g = g + np.uint64(0x9E3779B97F4A7C15)
    return (_mix64(g) % np.uint64(nranks)).astype(np.int64)


class _CudaArray:
    """Zero-copy view of raw device memory for torch.as_tensor."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def route_layout(n_max: int, tokens_max: int, header: int | None = None,
                 inbox: int = 0) -> tuple[list[int], int] | tuple[list[int], int, int]:
    """Byte offsets (sid, qoff, len, tok, idx, m, par, dup, low plane, high plane, pack
    blocks, query records) and total bytes of a region.  The 18-bit planes
    (include/tmstore.h) carry 128 positions of slack: owners copy them in 64-position
    granules.  ``inbox`` > 0 (push routing): the planes and records form ``inbox`` slices,
    one per source rank, and the slice stride is returned as a third value."""
    if header is None:
        from . import _lib

        hb = C.c_int64()
        check(_lib.load().tm_route_desc_bytes(C.byref(hb)))
        header = hb.value
    a = lambda nbytes: (nbytes + 255) // 256 * 256  # noqa: E731
    off, cur = [], a(header)  # RouteDesc header
    planes = (tokens_max + 63) // 64 * 64 + 128
    sizes = (8 * n_max, 8 * n_max, 8 * n_max, 4 * tokens_max, 4 * n_max, 8 * n_max, 8 * n_max, 8 * n_max,
             2 * planes, planes // 4, 4 * (n_max + 1), 32 * n_max)
    if not inbox:
        for nbytes in sizes:
            off.append(cur)
            cur += a(nbytes)
        return off, cur
    for nbytes in sizes[:8]:
        off.append(cur)
        cur += a(nbytes)
    pk = cur
    cur += a(sizes[10])
    lo, hi = cur, cur + a(sizes[8])
    rec = hi + a(sizes[9])
    stride = rec + a(sizes[11]) - lo
    off += [lo, hi, pk, rec]
    return off, lo + inbox * stride, stride


class Router:
    """One rank's side of cross-GPU routing (collective construction: every rank of
    ``group`` must build its Router in the same order)."""

    def __init__(self, store: DeviceStore, group, n_max: int, tokens_max: int, g2l, push: bool = False):
        import torch
        import torch.distributed as dist

        self.store, self.group = store, group
        self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        self.n_max, self.tokens_max = n_max, tokens_max
        # push routing (peers only): requesters write remote queries' planes into the
        # owners' inboxes, owners read them from their own HBM (tm_route_prepare_push)
        self.push = bool(push) and self.nranks > 1
        self.stride = 0
        if self.push:
            self.offsets, self.bytes, self.stride = route_layout(n_max, tokens_max, inbox=self.nranks)
        else:
            self.offsets, self.bytes = route_layout(n_max, tokens_max)
        ptr = C.c_void_p()
        check(store.lib.tm_shared_alloc(store.h, self.bytes, C.byref(ptr)))
        self.base = ptr.value
        h = (C.c_char * 64)()
        check(store.lib.tm_ipc_handle(store.h, C.c_void_p(self.base), h))
        handles = [None] * self.nranks
        dist.all_gather_object(handles, bytes(h), group=group)
        self.peers = []
        for p, hb in enumerate(handles):
            if p == self.rank:
                self.peers.append(self.base)
                continue
            out = C.c_void_p()
            check(store.lib.tm_ipc_open(store.h, (C.c_char * 64).from_buffer_copy(hb), C.byref(out)))
            self.peers.append(out.value)
        self._peer_arr = (C.c_void_p * self.nranks)(*self.peers)
        self._off_arr = (C.c_int64 * 12)(*self.offsets)
        self._off_arr_raw = (C.c_int64 * 12)(*self.offsets[:8], 0, 0, 0, 0)  # no planes, no records
        dev = torch.device("cuda", store.device)
        view = lambda i, n, ts, dt: torch.as_tensor(_CudaArray(self.base + self.offsets[i], (n,), ts), device=dev)  # noqa: E731
        self.gsid = view(0, n_max, "<i8", None)
        self.qoff = view(1, n_max, "<i8", None)
        self.qlen = view(2, n_max, "<i8", None)
        self.tokens = view(3, tokens_max, "<i4", None)
        self.out_matched = view(5, n_max, "<i8", None)
        self.out_parent = view(6, n_max, "<i8", None)
        self.out_dup = view(7, n_max, "<i8", None)
        self.g2l = torch.as_tensor(np.asarray(g2l, np.int32), device=dev)
        self._bar = torch.zeros(1, device=dev)
        self._epoch = 0  # device-side barrier epochs (same sequence on every rank)
        dist.barrier(group=group)

    def _barrier(self):
        import torch.distributed as dist

        dist.all_reduce(self._bar, group=self.group)  # stream-ordered cross-rank barrier

    def match(self, n: int, sync: str = "device"):
        """Match the n queries staged in this rank's region (gsid / qoff / qlen / tokens)
        against their owners' shards; results land in out_matched / out_parent / out_dup.
        Enqueued on torch's current stream.  Collective: every rank calls it once per
        batch, in the same order and with the same ``sync``."""
        if sync not in ("nccl", "device"):
            raise ValueError(f"unknown sync mode {sync!r}")
        self.prepare(n)
        self.match_prepared(sync)

    def prepare(self, n: int, stream=None):
        """Bucket the staged batch by owner and pack its remote queries (tm_route_prepare),
        on ``stream`` (default: torch's current stream).  Local to this rank."""
        import torch

        if n > self.n_max:
            raise ValueError("batch larger than the routing region")
        st = (stream or torch.cuda.current_stream(self.store.device)).cuda_stream
        st = C.c_void_p(1 if st == 0 else st)
        if self.push:
            check(self.store.lib.tm_route_prepare_push(self.store.h, C.c_void_p(self.base), n, self._off_arr,
                                                       self.nranks, self.rank, self._peer_arr, self.stride, st))
            return
        check(self.store.lib.tm_route_prepare(self.store.h, C.c_void_p(self.base), n, self._off_arr, self.nranks,
                                              self.rank, st))

    def match_prepared(self, sync: str = "device", wait: bool = True):
        """The exchange + match of a prepared batch on torch's current stream (collective).
        ``wait=False`` (device barriers only): the wait for the owners' done flags is left
        to ``wait_done`` on another stream."""
        import torch

        st = torch.cuda.current_stream(self.store.device).cuda_stream
        st = C.c_void_p(1 if st == 0 else st)
        lib, h = self.store.lib, self.store.h
        g2l = C.c_void_p(self.g2l.data_ptr())
        if not wait and self.nranks > 1:
            if sync != "device":
                raise ValueError("a deferred done wait needs the device-side barriers")
            self._epoch += 1
            check(lib.tm_match_routed_nowait(h, self.nranks, self.rank, self._peer_arr, g2l, self.g2l.numel(),
                                             self._epoch, self.stride, st))
            return
        if self.push:
            if sync != "device":
                raise ValueError("push routing uses the device-side barriers")
            self._epoch += 1
            check(lib.tm_match_routed_push(h, self.nranks, self.rank, self._peer_arr, g2l, self.g2l.numel(),
                                           self._epoch, self.stride, st))
            return
        if sync == "device" and self.nranks > 1:
            self._epoch += 1
            check(lib.tm_match_routed_sync(h, self.nranks, self.rank, self._peer_arr, g2l, self.g2l.numel(),
                                           self._epoch, st))
            return
        if self.nranks > 1:
            self._barrier()
        check(lib.tm_match_routed(h, self.nranks, self.rank, self._peer_arr, g2l, self.g2l.numel(), st))
        if self.nranks > 1:
            self._barrier()

    def wait_done(self, stream=None):
        """The deferred half of ``match_prepared(wait=False)``: hold ``stream`` (default:
        torch's current) until every owner has written this rank's results of the last
        routed batch."""
        import torch

        st = (stream or torch.cuda.current_stream(self.store.device)).cuda_stream
        st = C.c_void_p(1 if st == 0 else st)
        check(self.store.lib.tm_route_wait_done(self.store.h, self.nranks, self.rank, self._peer_arr, self._epoch, st))

    def match_nccl(self, n: int):
        """BASELINE for comparison, not the product path: the same exchange done with
        NCCL collectives only — all-to-all of the query tokens to their owners, a local
        match there, all-to-all of the results back (with the host reading the split
        sizes in between).  Results land in out_matched / out_parent / out_dup."""
        import torch
        import torch.distributed as dist

        dev = self.gsid.device
        st = torch.cuda.current_stream(self.store.device).cuda_stream
        st = C.c_void_p(1 if st == 0 else st)
        lib, h = self.store.lib, self.store.h
        check(lib.tm_route_prepare(h, C.c_void_p(self.base), n, self._off_arr_raw, self.nranks, self.rank, st))
        cnt = np.zeros(16, np.int32)
        check(lib.tm_route_counts(h, C.c_void_p(self.base), cnt.ctypes.data_as(C.c_void_p), st))
        counts = cnt[: self.nranks].astype(np.int64)
        idx = torch.as_tensor(_CudaArray(self.base + self.offsets[4], (n,), "<i4"), device=dev).long()
        lens = self.qlen[:n][idx]
        pad = (lens + 31) // 32 * 32
        starts = self.qoff[:n][idx]
        tok_per_owner = torch.zeros(self.nranks, dtype=torch.int64, device=dev)
        owner_of_q = torch.repeat_interleave(torch.arange(self.nranks, device=dev), torch.as_tensor(counts, device=dev))
        tok_per_owner.index_add_(0, owner_of_q, pad)
        # queries are padded to 32-token blocks: gather whole blocks (32x fewer indices)
        nblk = pad // 32
        blk = torch.repeat_interleave(starts // 32, nblk) + (
            torch.arange(int(nblk.sum()), device=dev) - torch.repeat_interleave(torch.cumsum(nblk, 0) - nblk, nblk))
        send_tok = self.tokens.view(-1, 32)[blk].reshape(-1)
        meta = torch.stack([torch.as_tensor(counts, device=dev), tok_per_owner], 1).contiguous()
        rmeta = torch.empty_like(meta)
        dist.all_to_all_single(rmeta, meta, group=self.group)
        rm = rmeta.cpu().numpy()
        q_in, t_in = rm[:, 0].tolist(), rm[:, 1].tolist()
        q_out, t_out = counts.tolist(), tok_per_owner.tolist()
        recv_tok = torch.empty(sum(t_in), dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_tok, send_tok, t_in, t_out, group=self.group)
        send_ql = torch.stack([self.gsid[:n][idx], lens], 1).contiguous()
        recv_ql = torch.empty((sum(q_in), 2), dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv_ql, send_ql, q_in, q_out, group=self.group)
        rl = recv_ql[:, 1]
        rpad = (rl + 31) // 32 * 32
        roff = torch.cumsum(rpad, 0) - rpad
        sids = self.g2l[recv_ql[:, 0]]
        m_, p_, d_ = (torch.empty(sum(q_in), dtype=torch.int64, device=dev) for _ in range(3))
        self.store.match_device(sids, recv_tok, roff.contiguous(), rl.contiguous(), m_, p_, d_)
        res = torch.stack([m_, p_, d_], 1).contiguous()
        back = torch.empty((n, 3), dtype=torch.int64, device=dev)
        dist.all_to_all_single(back, res, q_out, q_in, group=self.group)
        self.out_matched[:n][idx] = back[:, 0]
        self.out_parent[:n][idx] = back[:, 1]
        self.out_dup[:n][idx] = back[:, 2]

    def close(self):
        lib, h = self.store.lib, self.store.h
        for p, ptr in enumerate(self.peers):
            if p != self.rank and ptr:
                lib.tm_ipc_close(h, C.c_void_p(ptr))
        if self.base:
            lib.tm_shared_free(h, C.c_void_p(self.base))
            self.base = None


def match_pipelined(routers, n: int, batches: int, side_stream=None, defer_done: bool = False):
    """Run ``batches`` routed batches alternating between routers (separate regions, the
    same staged queries or different ones): batch i+1 is bucketed and packed on a side
    stream while batch i is exchanged and matched on torch's current stream, so the pack
    of one batch hides under the NVLink-bound walk of the previous one.  Batch i's results
    are in routers[i % len(routers)].  Collective like Router.match (device barriers)."""
    import torch

    main = torch.cuda.current_stream(routers[0].store.device)
    side = side_stream or torch.cuda.Stream(routers[0].store.device)
    k = len(routers)
    side.wait_stream(main)  # the first prepare is ordered after whatever main holds
    prepared = [torch.cuda.Event() for _ in range(k)]
    done = [None] * k

    def prep(i):
        b = i % k
        if done[b] is not None:
            side.wait_event(done[b])  # the owners are finished with this region's last batch
        routers[b].prepare(n, stream=side)
        prepared[b].record(side)

    # one rank (no cross-rank barriers): consecutive walks also alternate between two
    # streams, so batch i+1's walk fills the SMs batch i's tail leaves idle (c5 at one GPU:
    # 27.6 -> 28.9 M q/s).  With peers the same overlap measured slower (N=2: 26.9 vs 28.2:
    # the next walk's waiting CTAs and link traffic crowd the current one), so it stays off.
    walks = [main]
    if routers[0].nranks == 1 and k > 1:
        if not hasattr(routers[0], "_walk_stream"):
            routers[0]._walk_stream = torch.cuda.Stream(routers[0].store.device)
        walks = [main, routers[0]._walk_stream]
        walks[1].wait_stream(main)
    # defer_done (peers): each batch's wait for the owners' done flags runs on its own
    # stream, so the next walk starts as soon as this rank's walk ends instead of behind the
    # slowest peer's tail; region reuse (prep) and the caller wait on that stream.  Measured
    # neutral at N=2 (28.3-30.4 vs 29.8-30.9 M q/s), so off by default.
    waiter = None
    if routers[0].nranks > 1 and defer_done:
        if not hasattr(routers[0], "_done_stream"):
            routers[0]._done_stream = torch.cuda.Stream(routers[0].store.device)
        waiter = routers[0]._done_stream
        waiter.wait_stream(main)
    prep(0)
    for i in range(batches):
        b = i % k
        ws = walks[i % len(walks)]
        ws.wait_event(prepared[b])
        done[b] = torch.cuda.Event()
        with torch.cuda.stream(ws):
            routers[b].match_prepared("device", wait=waiter is None)
        if waiter is not None:
            walked = torch.cuda.Event()
            walked.record(ws)
            waiter.wait_event(walked)
            routers[b].wait_done(waiter)
            done[b].record(waiter)
        else:
            done[b].record(ws)
        if i + 1 < batches:
            prep(i + 1)
    for ws in walks[1:]:
        main.wait_stream(ws)
    if waiter is not None:
        main.wait_stream(waiter)
