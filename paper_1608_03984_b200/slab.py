"""x-slab decomposition of the acoustic step across ranks with a per-step halo
exchange.

The reference splits the grid into x-slabs for its worker threads
(/root/reference/pkg/src/fdroof/kernel.py:190-217, spans i*nx//n ..
(i+1)*nx//n) and all slabs read one shared padded array.  Across GPUs each
rank holds only its slab plus `r` ghost planes on every internal face (none
on the global faces, where the kernels' zero fill is the reference halo):

* every step runs the unchanged single-GPU kernels over the local array; the
  owned planes' stencils reach at most r planes, into the ghosts, so they are
  exact; the ghost planes' own updates are wrong and are discarded;
* then the r owned boundary planes of the new level go to each neighbour and
  its planes overwrite the local ghosts (one exchange step per time step; x is
  the slowest axis, so every message is one contiguous block of the level);
* the source is injected by its owner only, receivers are recorded by their
  owners (traces gathered back into global order).

Off-grid (trilinear) positions: the source goes to every slab whose owned
planes hold one of its corners (a corner on a ghost plane is overwritten by
the exchange).  A receiver belongs to the slab owning its base plane floor(x);
its upper corner plane may be the first ghost plane, which is sampled inside
the step, before the exchange.  With ghost width r + 1 that plane's update is
exact (its stencil stays within the ghosts, its previous level was exchanged
the step before), so off-grid receivers need `slab_halo(cfg)` = r + 1 ghost
planes.  Local positions are pos - gx0, exact in float64, so the trilinear
weights are unchanged.

The result is bit-identical to the single-grid run: the same arithmetic on the
same values at every owned point.  `SlabPlan` and the exchange are plain host
logic (tests/test_slab.py runs them with the numpy oracle on gloo ranks);
`run_slab` is the multi-process GPU path (NCCL point-to-point of plane blocks
over NVLink); `run_slabs` drives every slab of one process through the
library's own exchange (fdr_acoustic_slabs_run: boundary planes first, peer
copies into the neighbours' ghost planes overlapped with the interior planes).
"""

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ValidationError
from .kernel import KernelConfig, OffGridReceivers, OffGridSource, Receivers, Source, Sponge


@dataclass(frozen=True)
class SlabPlan:
    """The split of nx planes into n_slabs x-slabs with `halo` ghost planes."""

    nx: int
    n_slabs: int
    halo: int

    def __post_init__(self):
        if self.n_slabs < 1 or self.halo < 1 or self.nx < 1:
            raise ValidationError("need nx, n_slabs and halo >= 1")
        for i in range(self.n_slabs):
            x0, x1 = self.span(i)
            if self.n_slabs > 1 and x1 - x0 < self.halo:
                raise ValidationError(f"slab {i} owns {x1 - x0} planes < halo {self.halo}: "
                                      f"too many slabs for nx={self.nx}")
            gx0, gx1 = self.local_range(i)
            if gx1 - gx0 < 2 * self.halo + 1:
                raise ValidationError(f"slab {i} ({gx1 - gx0} planes with ghosts) is thinner "
                                      f"than the stencil (2r+1 = {2 * self.halo + 1})")

    def span(self, i: int):
        """Owned global planes [x0, x1) of slab i (kernel.py:190-217 split)."""
        return i * self.nx // self.n_slabs, (i + 1) * self.nx // self.n_slabs

    def ghosts(self, i: int):
        """Ghost planes below and above slab i (internal faces only)."""
        return (self.halo if i > 0 else 0), (self.halo if i < self.n_slabs - 1 else 0)

    def local_range(self, i: int):
        """Global planes [gx0, gx1) held by slab i, ghosts included."""
        (x0, x1), (lo, hi) = self.span(i), self.ghosts(i)
        return x0 - lo, x1 + hi

    def owned_local(self, i: int) -> slice:
        """The owned planes within slab i's local array."""
        x0, x1 = self.span(i)
        lo = self.ghosts(i)[0]
        return slice(lo, lo + x1 - x0)

    def messages(self, i: int):
        """(peer, send planes, recv planes) of slab i's exchange, local plane
        ranges [a, b): r owned boundary planes out, r ghost planes in."""
        own, r = self.owned_local(i), self.halo
        out = []
        if i > 0:
            out.append((i - 1, (own.start, own.start + r), (own.start - r, own.start)))
        if i < self.n_slabs - 1:
            out.append((i + 1, (own.stop - r, own.stop), (own.stop, own.stop + r)))
        return out


def slab_halo(cfg: KernelConfig) -> int:
    """Ghost planes per internal face that make the decomposition exact: the
    stencil radius, plus one for off-grid receivers (module docstring)."""
    return cfg.halo + (1 if isinstance(cfg.receivers, OffGridReceivers) else 0)


def slab_config(cfg: KernelConfig, plan: SlabPlan, i: int):
    """Slab i's KernelConfig (local dims, m / sponge slices, owner-only source
    and receivers) and the global indices of its receivers."""
    if plan.n_slabs > 1 and plan.halo < slab_halo(cfg):
        raise ValidationError(f"plan has {plan.halo} ghost planes; this config needs "
                              f"slab_halo(cfg) = {slab_halo(cfg)}")
    gx0, gx1 = plan.local_range(i)
    x0, x1 = plan.span(i)
    ny, nz = cfg.dims[1], cfg.dims[2]
    m = cfg.m if np.isscalar(cfg.m) else np.ascontiguousarray(np.asarray(cfg.m)[gx0:gx1])
    sponge = None
    if cfg.sponge is not None:
        sponge = Sponge(cfg.sponge.x[gx0:gx1], cfg.sponge.y, cfg.sponge.z)
    source = None
    if isinstance(cfg.source, OffGridSource):
        px, py, pz = (float(c) for c in cfg.source.position)
        bx = int(np.floor(px))
        if bx + 1 >= x0 and bx < x1:  # a corner plane is owned here
            source = OffGridSource((px - gx0, py, pz), cfg.source.series)
    elif cfg.source is not None and x0 <= cfg.source.location[0] < x1:
        sx, sy, sz = cfg.source.location
        source = Source((sx - gx0, sy, sz), cfg.source.series)
    receivers, rec_index = None, np.zeros(0, dtype=np.int64)
    if cfg.receivers is not None:
        off = isinstance(cfg.receivers, OffGridReceivers)
        loc = cfg.receivers.positions if off else cfg.receivers.locations
        base = np.floor(loc[:, 0]) if off else loc[:, 0]
        mine = (base >= x0) & (base < x1)
        rec_index = np.nonzero(mine)[0]
        if rec_index.size:
            local = loc[mine].copy()
            local[:, 0] -= gx0
            receivers = OffGridReceivers(local) if off else Receivers(local)
    local = KernelConfig(order=cfg.order, dims=(gx1 - gx0, ny, nz), n_t=cfg.n_t, dt=cfg.dt, h=cfg.h,
                         m=m, source=source, receivers=receivers, sponge=sponge)
    return local, rec_index


def exchange(level, plan: SlabPlan, i: int, group=None, rank_of=None) -> None:
    """One halo exchange of slab i's level (a tensor whose dim 0 is the local
    x planes, CPU or CUDA) with torch.distributed point-to-point: r owned
    boundary planes to each neighbour, r ghost planes from it."""
    import torch.distributed as dist

    rank_of = rank_of or (lambda j: j)
    ops = []
    for peer, (sa, sb), (ra, rb) in plan.messages(i):
        ops.append(dist.P2POp(dist.isend, level[sa:sb].contiguous(), rank_of(peer), group))
        ops.append(dist.P2POp(dist.irecv, level[ra:rb], rank_of(peer), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def exchange_local(levels, plan: SlabPlan) -> None:
    """The same exchange for all slabs held by one process (levels[i] is slab
    i's level): plane-block copies, for single-device validation."""
    sends = []
    for i in range(plan.n_slabs):
        for peer, (sa, sb), _ in plan.messages(i):
            sends.append((i, peer, levels[i][sa:sb].clone()))
    for i, peer, block in sends:
        for back, _, (ra, rb) in plan.messages(peer):
            if back == i:
                levels[peer][ra:rb].copy_(block)


def run_slabs_local(cfg: KernelConfig, plan: SlabPlan, n_steps: Optional[int] = None,
                    device=None, variant: str = "auto"):
    """All slabs of `plan` on one GPU, stepped in lock step with local
    exchanges; returns (global final level as numpy, global traces or None).
    The single-device check of the decomposition (no cross-waiting kernels)."""
    from . import kernel as K

    n = cfg.n_t if n_steps is None else int(n_steps)
    parts = [slab_config(cfg, plan, i) for i in range(plan.n_slabs)]
    flds = [K.Wavefield.allocate(c.dims, c.halo, device) for c, _ in parts]
    for _ in range(n):
        for (c, _), f in zip(parts, flds):
            K.run(f, c, 1, variant=variant)
        exchange_local([f.grids[2] for f in flds], plan)
    return gather_local(cfg, plan, parts, flds)


def gather_local(cfg, plan, parts, flds):
    nx, ny, nz = cfg.dims
    out = np.zeros((nx, ny, nz), dtype=flds[0].numpy().dtype)
    for i, f in enumerate(flds):
        x0, x1 = plan.span(i)
        out[x0:x1] = f.numpy()[plan.owned_local(i)]
    traces = None
    if cfg.receivers is not None:
        rows = max(cfg.n_t, flds[0].it)
        traces = np.zeros((rows, cfg.receivers.count), dtype=out.dtype)
        for (c, idx), f in zip(parts, flds):
            if idx.size and f.traces is not None:
                t = f.traces.cpu().numpy()
                traces[: t.shape[0], idx] = t
    return out, traces


def run_slab(cfg: KernelConfig, plan: SlabPlan, rank: int, n_steps: Optional[int] = None,
             group=None, device=None, variant: str = "auto", fld=None):
    """Rank `rank`'s slab on its GPU for n_steps with an NCCL halo exchange
    after every step; returns (local Wavefield, local config, receiver
    indices).  Pass `fld` to continue from an existing local state."""
    from . import kernel as K

    n = cfg.n_t if n_steps is None else int(n_steps)
    local, rec_index = slab_config(cfg, plan, rank)
    if fld is None:
        fld = K.Wavefield.allocate(local.dims, local.halo, device)
    for _ in range(n):
        K.run(fld, local, 1, variant=variant)
        exchange(fld.grids[2], plan, rank, group)
    return fld, local, rec_index


def gather_slabs(fld, plan: SlabPlan, rank: int, dims, group=None):
    """The global final level on every rank (all_gather of the owned planes)."""
    import torch
    import torch.distributed as dist

    own = fld.interior(2)[plan.owned_local(rank)].contiguous()
    widths = [plan.span(i)[1] - plan.span(i)[0] for i in range(plan.n_slabs)]
    parts = [torch.empty((w,) + tuple(own.shape[1:]), dtype=own.dtype, device=own.device)
             for w in widths]
    dist.all_gather(parts, own, group=group)
    full = torch.cat(parts, 0)
    if tuple(full.shape) != tuple(dims):
        raise ValidationError("gathered slabs do not tile the grid")
    return full


def run_slabs(cfg: KernelConfig, plan: SlabPlan, devices=None, n_steps: Optional[int] = None):
    """All slabs of `plan` in one process through the library's exchange
    (fdr_acoustic_slabs_run): slab i on devices[i] (default: every slab on
    the current device), each step's boundary planes computed first and
    copied into the neighbours' ghost planes (cudaMemcpyPeerAsync; NVLink
    between devices) while the interior planes are computed.  On-grid source
    and receivers (ghost width r).  Returns (global final level as numpy,
    global traces or None), like run_slabs_local."""
    import ctypes

    import torch

    from . import _lib
    from . import kernel as K

    if isinstance(cfg.source, OffGridSource) or isinstance(cfg.receivers, OffGridReceivers):
        raise ValidationError("run_slabs takes on-grid sources and receivers (run_slab / "
                              "run_slabs_local take off-grid ones)")
    if plan.halo != cfg.halo:
        raise ValidationError(f"run_slabs needs ghost width r = {cfg.halo}, plan has {plan.halo}")
    n = cfg.n_t if n_steps is None else int(n_steps)
    ns = plan.n_slabs
    if devices is None:
        devices = [torch.cuda.current_device()] * ns
    if len(devices) != ns:
        raise ValidationError("one device per slab")
    parts = [slab_config(cfg, plan, i) for i in range(ns)]
    flds = [K.Wavefield.allocate(c.dims, c.halo, torch.device("cuda", d))
            for (c, _), d in zip(parts, devices)]
    if n == 0:
        return gather_local(cfg, plan, parts, flds)
    keep = [K.device_args(f, c, n) for (c, _), f in zip(parts, flds)]
    arr = (_lib.AcousticArgs * ns)(*keep)
    devs = (ctypes.c_int * ns)(*[int(d) for d in devices])
    streams = (ctypes.c_void_p * ns)(*[torch.cuda.current_stream(d).cuda_stream for d in devices])
    _lib.check(_lib.load().fdr_acoustic_slabs_run(arr, ns, devs, streams))
    for f in flds:
        g = f.grids
        f.grids = [g[n % 3], g[(1 + n) % 3], g[(2 + n) % 3]]
        f.it += n
    return gather_local(cfg, plan, parts, flds)
