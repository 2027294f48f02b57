"""Device-resident H_eff·ψ plans — the drop-in for blocks.py:503 build_plan
and dmrg.py:107 apply_plan.

``build_plan`` keeps the reference signature and returns a ``DevicePlan``;
``apply_plan(plan, psi, out)`` keeps ``out += H_eff psi`` semantics and
accepts either the reference's ``SuperblockWavefunction`` objects (host
blocks: one H2D of ψ, one D2H of σ) or CUDA tensors laid out like
``to_vector`` (no copies).  All arithmetic runs in the sm_100a library; there
is no CPU path.
"""

import ctypes

import numpy as np

from . import _lib
from .plan_input import PlanInput, compile_reference_plan

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def _stream_handle(stream=None, device=None):
    if torch is None or not torch.cuda.is_available():
        return None
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


class _on_device:
    """Make the plan's device current around a library call (the library
    allocates and launches on the current device)."""

    def __init__(self, device):
        self.ctx = torch.cuda.device(device) if device is not None else None

    def __enter__(self):
        if self.ctx is not None:
            self.ctx.__enter__()

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)


def _desc(pi, arena_l=None, arena_r=None, rank=0, world=1, workspace_doubles=0,
          keep_groups=False, dry_run=False):
    P = _lib.as_p
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    d = _lib.PlanDesc()
    d.ncomp = pi.ncomp
    d.nsite = pi.nsite
    d.site_qn = P(pi.site_qn, i32)
    d.target = P(pi.target, i32)
    d.nsec_l = int(pi.dim_l.shape[0])
    d.qn_l = P(pi.qn_l, i32)
    d.dim_l = P(pi.dim_l, i32)
    d.left_sign = P(pi.left_sign, dbl)
    d.nsec_r = int(pi.dim_r.shape[0])
    d.qn_r = P(pi.qn_r, i32)
    d.dim_r = P(pi.dim_r, i32)
    d.nops_l = int(pi.kind_l.shape[0])
    d.delta_l = P(pi.delta_l, i32)
    d.blk_off_l = P(pi.blk_off_l, i64)
    d.kind_l = P(pi.kind_l, i32)
    d.nops_r = int(pi.kind_r.shape[0])
    d.delta_r = P(pi.delta_r, i32)
    d.blk_off_r = P(pi.blk_off_r, i64)
    d.kind_r = P(pi.kind_r, i32)
    d.nrows = pi.nrows
    d.lop = P(pi.lop, i32)
    d.rop = P(pi.rop, i32)
    d.alpha = P(pi.alpha, dbl)
    d.e_l = P(pi.e_l, i32)
    d.site1_dst = P(pi.site1_dst, i32)
    d.site1_val = P(pi.site1_val, dbl)
    d.site2_dst = P(pi.site2_dst, i32)
    d.site2_val = P(pi.site2_val, dbl)
    d.arena_l = _lib.ptr(arena_l)
    d.arena_r = _lib.ptr(arena_r)
    d.workspace_doubles = int(workspace_doubles)
    d.rank = int(rank)
    d.world = int(world)
    d.keep_groups = int(bool(keep_groups))
    d.dry_run = int(bool(dry_run))
    return d


class PlanGroups:
    """The reference grouping (blocks.py:563-567) as flat arrays."""

    def __init__(self, group_psi, group_out, group_begin, member_row, member_scale):
        self.group_psi = group_psi
        self.group_out = group_out
        self.group_begin = group_begin
        self.member_row = member_row
        self.member_scale = member_scale

    def __len__(self):
        return int(self.group_psi.shape[0])


class DevicePlan:
    """Task list + work list of one H_eff on one rank (sdmrg_plan_build).

    ``dry_run=True`` runs task generation only (no device), which is what
    the CPU test-suite uses to check grouping parity with the reference.
    """

    def __init__(self, pi, device=None, rank=0, world=1, workspace_doubles=0,
                 keep_groups=False, dry_run=False, arena_l=None, arena_r=None,
                 empty_arenas=False):
        """``empty_arenas``: the plan allocates zeroed padded arenas that the
        caller fills in place (``padded_arena``) — for operator sets too large
        to hold a dense copy beside the padded one."""
        lib = _lib.load()
        self.pi = pi.normalized()
        self.rank, self.world = int(rank), int(world)
        self.dry_run = bool(dry_run)
        self.device = None
        self.arena_l = self.arena_r = None
        if not dry_run:
            if torch is None or not torch.cuda.is_available():
                raise _lib.LibraryError("DevicePlan needs a CUDA device (no CPU fallback)")
            dev = torch.device(device if device is not None else "cuda")
            if dev.index is None:
                dev = torch.device("cuda", torch.cuda.current_device())
            self.device = dev
            if not empty_arenas:
                self.arena_l = arena_l if arena_l is not None else \
                    torch.from_numpy(self.pi.arena_l).to(self.device)
                self.arena_r = arena_r if arena_r is not None else \
                    torch.from_numpy(self.pi.arena_r).to(self.device)
        self._desc = _desc(self.pi, self.arena_l, self.arena_r, rank, world,
                           workspace_doubles, keep_groups, dry_run)
        handle = ctypes.c_void_p()
        with _on_device(self.device):
            _lib.check(lib.sdmrg_plan_build(ctypes.byref(self._desc), ctypes.byref(handle)))
        self._h = handle
        # the library repacked the arenas into plan-owned padded memory: the
        # caller's (or our temporary device) copies are no longer referenced
        self.arena_l = self.arena_r = None
        self._desc.arena_l = self._desc.arena_r = None
        st = _lib.PlanStats()
        _lib.check(lib.sdmrg_plan_stats_get(self._h, ctypes.byref(st)))
        self.stats = st.as_dict()
        nk = self.stats["psi_keys"]
        keys = np.zeros((nk, 4), dtype=np.int32)
        offs = np.zeros(nk + 1, dtype=np.int64)
        _lib.check(lib.sdmrg_plan_layout(self._h, _lib.as_p(keys, ctypes.c_int32),
                                         _lib.as_p(offs, ctypes.c_int64)))
        self.keys = keys
        self.offsets = offs
        self.keep_groups = keep_groups
        self.counter = None     # backend.counter of the drop-in apply_plan

    # reference-facing attributes (blocks.py:495 EffectiveHamiltonianPlan)
    @property
    def flops(self):
        return self.stats["ref_flops"]

    @property
    def psi_size(self):
        return self.stats["psi_size"]

    def groups(self):
        if not self.keep_groups:
            raise ValueError("plan built without keep_groups")
        g = self.stats["groups"]
        m = self.stats["members"]
        gp = np.zeros(g, np.int32)
        go = np.zeros(g, np.int32)
        gb = np.zeros(g + 1, np.int64)
        mr = np.zeros(m, np.int64)
        ms = np.zeros(m, np.float64)
        P = _lib.as_p
        _lib.check(_lib.load().sdmrg_plan_groups(
            self._h, P(gp, ctypes.c_int32), P(go, ctypes.c_int32), P(gb, ctypes.c_int64),
            P(mr, ctypes.c_int64), P(ms, ctypes.c_double)))
        return PlanGroups(gp, go, gb, mr, ms)

    def padded_arena(self, side):
        """(CUDA tensor view of the plan-owned padded arena, offsets[nops, nsec])
        for side 'l' or 'r' (sdmrg_plan_arena).  The view aliases plan memory:
        valid only while the plan lives; call ``invalidate()`` after writing
        through it once the plan has been applied."""
        k = {"l": 0, "r": 1}[side]
        nops = self.pi.kind_l.shape[0] if k == 0 else self.pi.kind_r.shape[0]
        nsec = self.pi.dim_l.shape[0] if k == 0 else self.pi.dim_r.shape[0]
        base = ctypes.c_void_p()
        size = ctypes.c_int64()
        offs = np.zeros((nops, nsec), np.int64)
        _lib.check(_lib.load().sdmrg_plan_arena(self._h, k, ctypes.byref(base),
                                                ctypes.byref(size),
                                                _lib.as_p(offs, ctypes.c_int64)))

        class _View:  # zero-copy device view (CUDA array interface)
            __cuda_array_interface__ = {"shape": (int(size.value),), "typestr": "<f8",
                                        "data": (int(base.value or 0), False), "version": 3}
        view = torch.as_tensor(_View(), device=self.device)
        return view, offs

    def diagonal(self, out=None):
        """The diagonal of H_eff over this rank's ψ sectors (device vector in
        the to_vector layout; sdmrg_plan_diagonal) — the Davidson
        preconditioner.  Sum over ranks for the full diagonal."""
        if out is None:
            out = torch.empty(self.psi_size, dtype=torch.float64, device=self.device)
        with _on_device(self.device):
            _lib.check(_lib.load().sdmrg_plan_diagonal(self._h, out.data_ptr(),
                                                       _stream_handle(device=self.device)))
        return out

    def block_layout(self, side):
        """offsets[nops, nsec] of the operator blocks this plan holds in its
        padded arena for side 'l' / 'r' (-1: not held — blocks no ψ sector of
        this rank reads); available in dry runs too."""
        k = {"l": 0, "r": 1}[side]
        nops = self.pi.kind_l.shape[0] if k == 0 else self.pi.kind_r.shape[0]
        nsec = self.pi.dim_l.shape[0] if k == 0 else self.pi.dim_r.shape[0]
        offs = np.zeros((nops, nsec), np.int64)
        _lib.check(_lib.load().sdmrg_plan_arena(self._h, k, None, None,
                                                _lib.as_p(offs, ctypes.c_int64)))
        return offs

    def shard(self):
        """Boolean mask over ψ keys: the input sectors this rank applies."""
        mine = np.zeros(self.stats["psi_keys"], np.int32)
        _lib.check(_lib.load().sdmrg_plan_shard(self._h, _lib.as_p(mine, ctypes.c_int32)))
        return mine.astype(bool)

    def empty_vector(self):
        return torch.empty(self.psi_size, dtype=torch.float64, device=self.device)

    def apply(self, psi, sigma=None, accumulate=False, stream=None):
        """sigma (+)= H_eff psi over this rank's shard (device tensors)."""
        if self.dry_run:
            raise _lib.LibraryError("dry-run plan cannot apply")
        if sigma is None:
            sigma = self.empty_vector()
            accumulate = False
        for v in (psi, sigma):
            if not (v.is_cuda and v.dtype == torch.float64 and v.is_contiguous()
                    and v.numel() == self.psi_size):
                raise ValueError("apply: vectors must be contiguous float64 CUDA tensors "
                                 f"of length {self.psi_size}")
        if psi.device != self.device or sigma.device != self.device:
            raise ValueError(f"apply: vectors must live on the plan's device {self.device}")
        with _on_device(self.device):
            _lib.check(_lib.load().sdmrg_plan_apply(
                self._h, psi.data_ptr(), sigma.data_ptr(), int(bool(accumulate)),
                _stream_handle(stream, self.device)))
        if self.counter is not None:   # reference accounting (sbmm4s.py:190 via gemm.py:22)
            self.counter.count(multiplies=2 * self.stats["groups"], flops=self.flops)
        return sigma

    __call__ = apply

    def invalidate(self):
        """The arenas changed in place: the next apply re-forms the operator
        pre-sums (sdmrg_plan_invalidate)."""
        _lib.check(_lib.load().sdmrg_plan_invalidate(self._h))

    def set_timing(self, enable=True):
        """Record CUDA events around every engine launch of later applies."""
        _lib.check(_lib.load().sdmrg_plan_set_timing(self._h, int(bool(enable))))

    def last_timing(self):
        """Per-phase device ms, executed FLOPs and algorithmic bytes of the last
        apply: phase 0 left-operator pre-summation, 1 T = A R^T, 2 σ += Lsum T,
        3 split-K partial sums into σ."""
        ms = (ctypes.c_double * 4)()
        fl = (ctypes.c_int64 * 4)()
        by = (ctypes.c_int64 * 4)()
        _lib.check(_lib.load().sdmrg_plan_timing(self._h, ms, fl, by))
        return list(ms), list(fl), list(by)

    def close(self):
        if getattr(self, "_h", None):
            with _on_device(self.device):
                _lib.load().sdmrg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_plan(model, table, left_store, right_store, psi_struct, aux_mats=None,
               rank=0, world=1, keep_groups=False):
    """Drop-in for blocks.py:503 build_plan: same arguments, device plan out."""
    pi = compile_reference_plan(model, table, left_store, right_store, psi_struct,
                                aux_mats)
    plan = DevicePlan(pi, rank=rank, world=world, keep_groups=keep_groups)
    plan.psi_struct = psi_struct
    return plan


def apply_plan(plan, psi, out, pool=None, arenas=None, backend=None, locks=None):
    """Drop-in for dmrg.py:107 apply_plan: ``out += H_eff psi``.

    With reference ``SuperblockWavefunction`` arguments the ψ blocks are
    copied to the device once, σ comes back once (the e2e path); with CUDA
    tensors nothing leaves the device.  ``pool``/``arenas``/``backend``/
    ``locks`` are accepted for signature compatibility: the device plan owns
    its scheduling (persistent CTAs) and needs no per-sector locks because
    every σ tile has exactly one owner.
    """
    if backend is not None and getattr(backend, "counter", None) is not None:
        plan.counter = backend.counter      # driver.py:138 reads counter.snapshot()[2]
    if torch is not None and isinstance(psi, torch.Tensor):
        return plan.apply(psi, out, accumulate=True)
    vec = psi.to_vector()
    dpsi = torch.from_numpy(np.ascontiguousarray(vec)).to(plan.device)
    dout = torch.from_numpy(np.ascontiguousarray(out.to_vector())).to(plan.device)
    plan.apply(dpsi, dout, accumulate=True)
    res = dout.cpu().numpy()
    pos = 0
    for key in out.keys:
        shape = out.block_shape(key)
        n = shape[0] * shape[1]
        out.blocks[key][...] = res[pos:pos + n].reshape(shape)
        pos += n
    return out


apply_effective_hamiltonian = apply_plan
