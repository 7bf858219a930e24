"""Frequency-sharded multi-GPU solve: one process per GPU, torch.distributed
(NCCL over NVLink on B200; gloo for the CPU tests) for the plumbing, the per-rank kernels through
the shard-level C-ABI (`fpc_shard_*`).

Layouts (G ranks, N = Nt*Ns, H = Nt/2 + 1):
  * Krylov vectors: time-sharded, rank g owns time blocks [g*Nt/G, (g+1)*Nt/G) (contiguous).
  * matvec (all_at_once.hpp:33-55): local, after an all-gather of every rank's last two blocks
    (the BDF2 halo of the next rank).
  * PC apply (alpha_circulant.hpp:137-199), the reference ordering:
      all-to-all time -> space columns; time FFT (local columns); all-to-all space -> frequency rows;
      tau solves (local rows, alpha_circulant.hpp:160 -- the independent PinT work);
      all-to-all back to space; inverse time FFT; all-to-all back to time.
  * PC apply, commuted ordering (ordering="commuted", 1D and 2D): DST of every local time
    level; all-to-all time -> space columns; per-column time solve (FFT, divide, inverse FFT);
    all-to-all back to time; DST of every local time level -- two all-to-alls instead of four,
    real-valued in flight, rounding-level difference from the reference ordering.
  * Gram-Schmidt dots / norms: local partials + all_reduce (krylov.hpp:116-131).
Every rank runs the same host-side Hessenberg/Givens recurrence on the reduced values.

The local kernels are an object with the methods of `CudaShardKernels`; tests/dist_cpu_kernels.py
provides a numpy implementation so the communication logic runs under gloo on CPU.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N


def split_counts(total: int, parts: int) -> list[int]:
    return [total // parts + (1 if g < total % parts else 0) for g in range(parts)]


def offsets(counts: list[int]) -> list[int]:
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += c
    return out


@dataclass
class ShardReport:
    converged: bool = False
    iterations: int = 0
    restarts: int = 0
    residual_history: list = field(default_factory=list)
    final_relative_residual: float = 0.0
    true_relative_residual: float = 0.0
    reorthogonalizations: int = 0


class CudaShardKernels:
    """Per-rank kernels on CUDA tensors through the shard-level C-ABI."""

    def __init__(self, op, plan):
        self.op, self.plan, self.lib = op, plan, op.lib
        self.ctx = op.ctx
        self.device = torch.device("cuda", op.ctx.device)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def empty(self, n, complex_=False):
        return torch.empty(n, dtype=torch.complex128 if complex_ else torch.float64, device=self.device)

    def matvec(self, buf, nt_local, koff, halo):
        ns = self.op.n_space()
        y = self.empty(nt_local * ns)
        vptr = buf.data_ptr() + (2 * ns * 8 if halo else 0)
        N.check(self.lib.fpc_shard_matvec(self.op.h, C.c_void_p(vptr), self._p(y), nt_local, koff))
        return y

    def time_fwd(self, cols, ns_local, s_in):
        Z = self.empty((self.plan.n_time // 2 + 1) * ns_local, True)
        N.check(self.lib.fpc_shard_time_fwd(self.plan.h, self._p(cols), self._p(Z), ns_local, float(s_in)))
        return Z

    def tau(self, Zrows, row0, nrows, forward=False):
        N.check(self.lib.fpc_shard_tau(self.plan.h, self._p(Zrows), row0, nrows, int(forward)))

    def time_inv(self, Z, ns_local):
        z = self.empty(self.plan.n_time * ns_local)
        N.check(self.lib.fpc_shard_time_inv(self.plan.h, self._p(Z), self._p(z), ns_local))
        return z

    def dst_levels(self, v, nt_local, s_in):
        out = self.empty(v.numel())
        N.check(self.lib.fpc_shard_dst_levels(self.plan.h, self._p(v), self._p(out), nt_local, float(s_in)))
        return out

    def time_solve(self, cols, col0, ns_local, forward=False):
        z = self.empty(cols.numel())
        N.check(self.lib.fpc_shard_time_solve(self.plan.h, self._p(cols), self._p(z), col0, ns_local, int(forward)))
        return z

    def _ptrs(self, V):
        arr = (C.c_void_p * max(len(V), 1))(*[v.data_ptr() for v in V])
        return arr

    def dots(self, V, scales, w, with_norm):
        out = np.zeros(len(V) + 1)
        sc = np.ascontiguousarray(scales, dtype=np.float64)
        N.check(self.lib.fpc_shard_dots(self.ctx.h, self._ptrs(V), C.c_void_p(sc.ctypes.data), len(V),
                                        self._p(w), w.numel(), int(with_norm), C.c_void_p(out.ctypes.data)))
        return out[:len(V) + (1 if with_norm or not V else 0)]

    # device-resident variants: the partial sums stay on the GPU for an in-place NCCL all-reduce
    def dots_dev(self, V, scales, w, with_norm):
        cnt = len(V) + (1 if with_norm or not V else 0)
        out = torch.empty(max(cnt, 1), dtype=torch.float64, device=self.device)
        sc = np.ascontiguousarray(scales, dtype=np.float64)
        N.check(self.lib.fpc_shard_dots_dev(self.ctx.h, self._ptrs(V), C.c_void_p(sc.ctypes.data), len(V),
                                            self._p(w), w.numel(), int(with_norm), self._p(out)))
        return out[:cnt]

    def update_dev(self, V, coef, w):
        c = np.ascontiguousarray(coef, dtype=np.float64)
        out = torch.empty(1, dtype=torch.float64, device=self.device)
        N.check(self.lib.fpc_shard_update_dev(self.ctx.h, self._ptrs(V), C.c_void_p(c.ctypes.data), len(V),
                                              self._p(w), w.numel(), self._p(out)))
        return out

    def update(self, V, coef, w):
        c = np.ascontiguousarray(coef, dtype=np.float64)
        out = np.zeros(1)
        N.check(self.lib.fpc_shard_update(self.ctx.h, self._ptrs(V), C.c_void_p(c.ctypes.data), len(V),
                                          self._p(w), w.numel(), C.c_void_p(out.ctypes.data)))
        return float(out[0])

    def lincomb(self, V, coef):
        u = self.empty(V[0].numel())
        c = np.ascontiguousarray(coef, dtype=np.float64)
        N.check(self.lib.fpc_shard_lincomb(self.ctx.h, self._ptrs(V), C.c_void_p(c.ctypes.data), len(V),
                                           self._p(u), u.numel()))
        return u

    def synchronize(self):
        self.ctx.synchronize()

    # peer-store transport (kernels_p2p.cu)
    def alloc_shared(self, n_doubles):
        ptr = C.c_void_p()
        N.check(self.lib.fpc_device_alloc(self.ctx.h, max(8 * int(n_doubles), 16), C.byref(ptr)))
        return ptr.value

    def free_shared(self, ptr):
        self.lib.fpc_device_free(self.ctx.h, C.c_void_p(ptr))

    def ipc_handle(self, ptr) -> bytes:
        h = C.create_string_buffer(64)
        N.check(self.lib.fpc_ipc_get_handle(C.c_void_p(ptr), h))
        return h.raw

    def ipc_open(self, handle: bytes):
        ptr = C.c_void_p()
        N.check(self.lib.fpc_ipc_open(self.ctx.h, C.create_string_buffer(handle, 64), C.byref(ptr)))
        return ptr.value

    def ipc_close(self, ptr):
        self.lib.fpc_ipc_close(self.ctx.h, C.c_void_p(ptr))

    def tensor_at(self, ptr, n_doubles):
        """A float64 CUDA tensor over n doubles at a device pointer this object owns (zero copy)."""
        class _Buf:
            __cuda_array_interface__ = {"shape": (int(n_doubles),), "typestr": "<f8", "data": (int(ptr), False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_Buf(), device=self.device)

    def scatter_p2p(self, src, rows, cols, es, split_cols, dst_ptrs, off, stride, row_base, col_base):
        G = len(dst_ptrs)
        d = (C.c_void_p * G)(*dst_ptrs)
        o = (C.c_int * G)(*off)
        st = (C.c_int * G)(*stride)
        N.check(self.lib.fpc_shard_scatter_p2p(self.ctx.h, self._p(src), int(rows), int(cols), int(es),
                                               int(split_cols), d, o, st, G, int(row_base), int(col_base)))


class P2PTransport:
    """Receive buffers of the sharded PC apply's exchanges, one per exchange, mapped into every rank
    by CUDA IPC; an exchange is one peer-store kernel (fpc_shard_scatter_p2p: pack, NVLink transfer
    and unpack in one pass) followed by a stream-ordered barrier (one-element all_reduce on the same
    stream), replacing all_to_all_single and the copies around it.  Correct by construction for the
    buffer reuse: each exchange owns its buffer, and a rank rewrites a peer's buffer only after that
    peer has passed a later barrier, i.e. after its consumer kernel of the previous contents ran."""

    def __init__(self, kernels, group, G: int, rank: int, sizes: dict):
        self.k, self.group, self.G, self.rank = kernels, group, G, rank
        self.local, self.ptrs, self._opened = {}, {}, []
        for name, n in sizes.items():
            ptr = kernels.alloc_shared(n)
            self.local[name] = (ptr, int(n))
            handles = [None] * G
            if G > 1:
                dist.all_gather_object(handles, kernels.ipc_handle(ptr), group=group)
            ptrs = []
            for d in range(G):
                if d == rank:
                    ptrs.append(ptr)
                else:
                    q = kernels.ipc_open(handles[d])
                    self._opened.append(q)
                    ptrs.append(q)
            self.ptrs[name] = ptrs
        self._flag = torch.zeros(1, dtype=torch.float64, device=kernels.device)
        self._lib_stream = torch.cuda.ExternalStream(kernels.ctx.stream_handle, device=kernels.device)

    def exchange(self, name, src, rows, cols, es, split_cols, off, stride, row_base, col_base):
        """Scatter src into every rank's `name` buffer; returns this rank's buffer (float64 view)
        once every rank's stores into it are complete (stream order)."""
        self.k.scatter_p2p(src, rows, cols, es, split_cols, self.ptrs[name], off, stride, row_base, col_base)
        if self.G > 1:
            # the barrier must be ordered behind the scatter kernel, i.e. enqueued on the library
            # context's stream (not whatever torch stream is current)
            with torch.cuda.stream(self._lib_stream):
                dist.all_reduce(self._flag, group=self.group)
        ptr, n = self.local[name]
        return self.k.tensor_at(ptr, n)

    def close(self):
        """Unmap the peers' buffers, then -- only after every rank has unmapped this rank's buffers
        (barrier) -- free the exported ones: freeing an IPC-exported allocation while an importer
        still maps it is undefined."""
        self.k.synchronize()
        for q in self._opened:
            self.k.ipc_close(q)
        self._opened = []
        self.k.synchronize()
        if self.G > 1 and dist.is_initialized():
            dist.barrier(group=self.group)
        for ptr, _ in self.local.values():
            self.k.free_shared(ptr)
        self.local = {}


class ShardedSolver:
    """Right-preconditioned GMRES (krylov.hpp:83-192, + GMRES(m) restarts) over G ranks."""

    def __init__(self, n_time: int, n_space: int, kernels, group=None, ordering: str = "reference",
                 transport: str = "nccl"):
        if ordering not in ("reference", "commuted"):
            raise ValueError("ShardedSolver: ordering must be 'reference' or 'commuted'")
        if transport not in ("nccl", "p2p"):
            raise ValueError("ShardedSolver: transport must be 'nccl' or 'p2p'")
        if transport == "p2p" and not isinstance(kernels, CudaShardKernels):
            raise ValueError("ShardedSolver: the p2p transport needs the CUDA shard kernels")
        self.transport = transport
        self.ordering = ordering
        self.k = kernels
        self.group = group
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if n_time % self.G:
            raise ValueError("ShardedSolver: n_time must be divisible by the number of ranks")
        self.nt, self.ns = n_time, n_space
        self.H = n_time // 2 + 1
        self.nt_loc = n_time // self.G
        self.cs = split_counts(n_space, self.G)
        self.co = offsets(self.cs)
        self.hs = split_counts(self.H, self.G)
        self.ho = offsets(self.hs)
        self.koff = self.rank * self.nt_loc
        # CUDA kernels: Gram-Schmidt partials reduced on the device (one host read per reduction)
        self._dev_reduce = hasattr(kernels, "dots_dev")
        if self._dev_reduce:
            self._lib_stream = torch.cuda.ExternalStream(kernels.ctx.stream_handle, device=kernels.device)
        self.p2p = None
        if transport == "p2p":
            r = self.rank
            self.p2p = P2PTransport(kernels, group, self.G, r, {
                "cols": n_time * self.cs[r],              # time -> space columns [Nt][cs_r]
                "rows": 2 * self.hs[r] * n_space,         # space -> frequency rows [hs_r][Ns] complex
                "Z": 2 * self.H * self.cs[r],             # frequency -> space [H][cs_r] complex
                "w": self.nt_loc * n_space})              # space -> time [nt_loc][Ns]

    def close(self):
        if self.p2p is not None:
            self.p2p.close()
            self.p2p = None

    # peer-store versions of the exchanges (transport="p2p")
    def _x_time_to_space(self, v_loc):
        r = self.rank
        return self.p2p.exchange("cols", v_loc, self.nt_loc, self.ns, 1, True, self.co, self.cs,
                                 r * self.nt_loc, 0)

    def _x_space_to_time(self, z):
        r = self.rank
        return self.p2p.exchange("w", z, self.nt, self.cs[r], 1, False, [d * self.nt_loc for d in range(self.G)],
                                 [self.ns] * self.G, 0, self.co[r])

    # ------------------------------------------------------------------ collectives
    def _a2a(self, send_chunks, recv_sizes, like):
        """all_to_all of flat float64 views; send_chunks[d] goes to rank d."""
        if self.G == 1:
            return [send_chunks[0]]
        real = lambda t: torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)
        f = 2 if like.is_complex() else 1
        inp = torch.cat([real(c.contiguous()) for c in send_chunks])
        out = torch.empty(sum(recv_sizes) * f, dtype=torch.float64, device=inp.device)
        dist.all_to_all_single(out, inp, output_split_sizes=[s * f for s in recv_sizes],
                               input_split_sizes=[c.numel() * f for c in send_chunks], group=self.group)
        parts, o = [], 0
        for s in recv_sizes:
            p = out[o:o + s * f]
            parts.append(torch.view_as_complex(p.view(-1, 2)) if f == 2 else p)
            o += s * f
        return parts

    def _allreduce(self, arr: np.ndarray) -> np.ndarray:
        if self.G == 1:
            return arr
        dev = self.k.device if hasattr(self.k, "device") else torch.device("cpu")
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def _allreduce_dev(self, t):
        """In-place all-reduce of device partials, enqueued on the library stream behind the kernels
        that produced them; one host read of the sum."""
        if self.G > 1:
            with torch.cuda.stream(self._lib_stream):
                dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def _dots(self, V, sc, w, with_norm):
        if self._dev_reduce:
            return self._allreduce_dev(self.k.dots_dev(V, sc, w, with_norm))
        return self._allreduce(self.k.dots(V, sc, w, with_norm))

    def _update(self, V, coef, w):
        if self._dev_reduce:
            return float(self._allreduce_dev(self.k.update_dev(V, coef, w))[0])
        return float(self._allreduce(np.array([self.k.update(V, coef, w)]))[0])

    def _peer(self, group_rank):
        return dist.get_global_rank(self.group, group_rank) if self.group is not None else group_rank

    # ------------------------------------------------------------------ operators
    def matvec(self, v_loc):
        ns, G, r = self.ns, self.G, self.rank
        halo = None
        if G > 1:
            if self.nt_loc < 2:
                raise ValueError("ShardedSolver: need at least two time blocks per rank")
            # the BDF2 halo (the last two levels of rank r-1) point to point: send to r+1, receive from r-1
            tail = v_loc[(self.nt_loc - 2) * ns:].contiguous()
            ops = []
            if r + 1 < G:
                ops.append(dist.P2POp(dist.isend, tail, self._peer(r + 1), group=self.group))
            if r > 0:
                halo = torch.empty_like(tail)
                ops.append(dist.P2POp(dist.irecv, halo, self._peer(r - 1), group=self.group))
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if halo is not None:
            buf = torch.cat([halo, v_loc])
            return self.k.matvec(buf, self.nt_loc, self.koff, True)
        return self.k.matvec(v_loc, self.nt_loc, self.koff, False)

    def pc_apply(self, v_loc, s_in=1.0, forward=False):
        if self.ordering == "commuted":
            return self._pc_apply_commuted(v_loc, s_in, forward)
        G, r, ns, nt_loc = self.G, self.rank, self.ns, self.nt_loc
        if self.p2p is not None:
            cols = self._x_time_to_space(v_loc)
            Z = self.k.time_fwd(cols, self.cs[r], s_in)
            rows = self.p2p.exchange("rows", torch.view_as_real(Z).reshape(-1), self.H, self.cs[r], 2, False,
                                     self.ho, [ns] * G, 0, self.co[r])
            self.k.tau(torch.view_as_complex(rows.view(-1, 2)), self.ho[r], self.hs[r], forward)
            Zb = self.p2p.exchange("Z", rows, self.hs[r], ns, 2, True, self.co, self.cs, self.ho[r], 0)
            z = self.k.time_inv(torch.view_as_complex(Zb.view(-1, 2)), self.cs[r])
            return self._x_space_to_time(z).clone()  # the buffer is reused by the next apply
        V = v_loc.view(nt_loc, ns)
        # 1. time -> space columns
        parts = self._a2a([V[:, self.co[d]:self.co[d] + self.cs[d]] for d in range(G)],
                          [nt_loc * self.cs[r]] * G, v_loc)
        cols = torch.cat([p.view(nt_loc, self.cs[r]) for p in parts]).reshape(-1)
        # 2. time FFT on my columns -> half spectrum [H][cs]
        Z = self.k.time_fwd(cols, self.cs[r], s_in).view(self.H, self.cs[r])
        # 3. space -> frequency rows
        parts = self._a2a([Z[self.ho[d]:self.ho[d] + self.hs[d]] for d in range(G)],
                          [self.hs[r] * self.cs[s] for s in range(G)], Z)
        rows = torch.cat([p.view(self.hs[r], self.cs[s]) for s, p in enumerate(parts)], dim=1).contiguous()
        # 4. tau solves on my frequency rows
        self.k.tau(rows.view(-1), self.ho[r], self.hs[r], forward)
        # 5. frequency -> space
        parts = self._a2a([rows[:, self.co[d]:self.co[d] + self.cs[d]] for d in range(G)],
                          [self.hs[s] * self.cs[r] for s in range(G)], rows)
        Z = torch.cat([p.view(self.hs[s], self.cs[r]) for s, p in enumerate(parts)]).contiguous()
        # 6. inverse time FFT -> [Nt][cs]
        z = self.k.time_inv(Z.view(-1), self.cs[r]).view(self.nt, self.cs[r])
        # 7. space -> time
        parts = self._a2a([z[d * nt_loc:(d + 1) * nt_loc] for d in range(G)],
                          [nt_loc * self.cs[s] for s in range(G)], z)
        return torch.cat([p.view(nt_loc, self.cs[s]) for s, p in enumerate(parts)], dim=1).reshape(-1).contiguous()

    def _pc_apply_commuted(self, v_loc, s_in=1.0, forward=False):
        G, r, ns, nt_loc = self.G, self.rank, self.ns, self.nt_loc
        if self.p2p is not None:
            u = self.k.dst_levels(v_loc, nt_loc, s_in)
            z = self.k.time_solve(self._x_time_to_space(u), self.co[r], self.cs[r], forward)
            return self.k.dst_levels(self._x_space_to_time(z), nt_loc, 1.0)
        # 1. S on every local time level (no communication)
        u = self.k.dst_levels(v_loc, nt_loc, s_in).view(nt_loc, ns)
        # 2. time -> space columns
        parts = self._a2a([u[:, self.co[d]:self.co[d] + self.cs[d]] for d in range(G)],
                          [nt_loc * self.cs[r]] * G, u)
        cols = torch.cat([p.view(nt_loc, self.cs[r]) for p in parts]).reshape(-1)
        # 3. per spatial mode: time FFT, divide by (lambda_n - dt sigma_p), inverse FFT
        z = self.k.time_solve(cols, self.co[r], self.cs[r], forward).view(self.nt, self.cs[r])
        # 4. space -> time
        parts = self._a2a([z[d * nt_loc:(d + 1) * nt_loc] for d in range(G)],
                          [nt_loc * self.cs[s] for s in range(G)], z)
        w = torch.cat([p.view(nt_loc, self.cs[s]) for s, p in enumerate(parts)], dim=1).reshape(-1).contiguous()
        # 5. S on every local time level
        return self.k.dst_levels(w, nt_loc, 1.0)

    # ------------------------------------------------------------------ GMRES
    def _norm(self, w):
        return math.sqrt(float(self._dots([], [], w, True)[0]))

    def _inner(self, b, tol, max_iter, rep):
        """One unrestarted gmres_right (x0 = 0) on rhs b; returns x, steps, converged."""
        norm_b = self._norm(b)
        if norm_b == 0.0:
            return torch.zeros_like(b), 0, True
        V, sc = [b], [1.0 / norm_b]
        hcols, gc, gs, g = [], [], [], [norm_b]
        steps, conv = 0, False
        for j in range(max_iter):
            z = self.pc_apply(V[j], sc[j])
            w = self.matvec(z)
            nv = j + 1
            d = self._dots(V, sc, w, True)
            h = list(d[:nv]) + [0.0]
            norm_before = math.sqrt(d[nv])
            nw2 = self._update(V, [h[i] * sc[i] for i in range(nv)], w)
            norm_w = math.sqrt(nw2)
            if norm_w < 0.70710678118654752 * norm_before:  # krylov.hpp:123-130
                rep.reorthogonalizations += 1
                c2 = self._dots(V, sc, w, False)
                nw2 = self._update(V, [c2[i] * sc[i] for i in range(nv)], w)
                for i in range(nv):
                    h[i] += c2[i]
                norm_w = math.sqrt(nw2)
            h[j + 1] = norm_w
            for i in range(j):  # krylov.hpp:133-151
                hi, hi1 = h[i], h[i + 1]
                h[i] = gc[i] * hi + gs[i] * hi1
                h[i + 1] = -gs[i] * hi + gc[i] * hi1
            rad = math.hypot(h[j], h[j + 1])
            cs_ = h[j] / rad if rad > 0 else 1.0
            sn_ = h[j + 1] / rad if rad > 0 else 0.0
            gc.append(cs_)
            gs.append(sn_)
            h[j], h[j + 1] = rad, 0.0
            g.append(-sn_ * g[j])
            g[j] *= cs_
            hcols.append(h)
            steps = j + 1
            rel = abs(g[j + 1]) / norm_b
            rep.residual_history.append(rel)
            if rel <= tol:
                conv = True
                break
            if norm_w <= 1e-14 * max(1.0, norm_before):
                break
            V.append(w)
            sc.append(1.0 / norm_w)
        y = [0.0] * steps
        for i in range(steps - 1, -1, -1):
            s = g[i]
            for kk in range(i + 1, steps):
                s -= hcols[kk][i] * y[kk]
            y[i] = s / hcols[i][i]
        u = self.k.lincomb(V[:steps], [y[i] * sc[i] for i in range(steps)]) if steps else torch.zeros_like(b)
        return self.pc_apply(u), steps, conv

    def gmres(self, b_loc, tol=1e-9, max_iter=200, restart=0):
        rep = ShardReport()
        norm_b = self._norm(b_loc)
        if restart <= 0 or restart >= max_iter:
            x, steps, conv = self._inner(b_loc, tol, max_iter, rep)
            rep.iterations, rep.converged = steps, conv
        else:  # restart emulation, SURVEY §8(c) (same as oracle/fracpint_oracle.c)
            x = torch.zeros_like(b_loc)
            r = b_loc.clone()
            budget, total, conv = max_iter, 0, False
            while budget > 0:
                norm_r = self._norm(r)
                if norm_r == 0.0:
                    conv = True
                    break
                h0 = len(rep.residual_history)
                d, steps, c = self._inner(r, tol * norm_b / norm_r, min(restart, budget), rep)
                for i in range(h0, len(rep.residual_history)):
                    rep.residual_history[i] *= norm_r / norm_b
                x = x + d
                total += steps
                budget -= steps
                if c:
                    conv = True
                    break
                if steps == 0:
                    break
                rep.restarts += 1
                r = b_loc - self.matvec(x)
            rep.iterations, rep.converged = total, conv
        rep.final_relative_residual = rep.residual_history[-1] if rep.residual_history else 1.0
        if norm_b == 0.0:
            rep.true_relative_residual = 0.0
        else:
            res = b_loc - self.matvec(x)
            rep.true_relative_residual = self._norm(res) / norm_b
        return x, rep
