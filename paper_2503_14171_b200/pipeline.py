"""Batched multi-view render + upscale pipeline (the throughput path).

``ViewPipeline`` renders many camera views of one scene at W x H and
gradient-upscales each to the output size, reusing per-slot workspaces so the
steady state allocates nothing and never synchronises the host per view.  Each
view is exactly ``upscale_spline(render_forward(scene, W, H, view=v), factor)``
(tests/test_gpu_pipeline.py checks this), i.e. the reference's
``render_forward`` + ``upscale_spline`` (raster_forward.py:152, spline.py:162)
on the view scene of ``scenes.view_scene``.

Pair-buffer capacity is calibrated once per view set (untimed); a sticky
device flag records any overflow and ``check()`` raises on it, so an
under-sized buffer can never silently drop splats.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .core import DimensionError
from .device import to_device
from .raster_forward import BIN_COUNT_ONLY, Frame, GradientImage, make_view
from .spline import check_output, output_size, upscale_plan

STAGES = ("prepare", "bin", "raster", "fixup", "upscale")
DEFER_FIXUP = 2   # splat_rasterize flag (SPLAT_RASTER_DEFER_FIXUP): the fix-up runs as its own call


class _Slot:
    def __init__(self, pipe, stream):
        self.stream = stream
        self.frame = Frame(pipe.scene.n, pipe.width, pipe.height, pipe.capacity, pipe.scene.device)
        self.img = GradientImage.empty(pipe.width, pipe.height, pipe.scene.device)
        self.out = [torch.empty((pipe.out_h, pipe.out_w, 3), dtype=torch.float32,
                                device=pipe.scene.device) for _ in range(2)]
        self.copied = [None, None]   # events: D2H of out[k] finished
        self.flip = 0
        self.gimg = self.img.c_gimg()


class ViewPipeline:
    BATCHED = True   # one splat_render_views call per batch (False: the per-view ABI calls)
    def __init__(self, scene, width: int, height: int, *, factor: float = 4.0, out_size=None,
                 slots: int = 1, capacity: int | None = None, views_for_capacity=None):
        self.scene = to_device(scene)
        self.width, self.height = int(width), int(height)
        if out_size is None:
            self.out_w, self.out_h = output_size(self.width, self.height, factor)
        else:
            self.out_w, self.out_h = (int(v) for v in out_size)
        self.lib = _lib.load()
        if capacity is None:
            capacity = self.calibrate(views_for_capacity or [None])
        self.capacity = int(capacity)
        self.nslots = slots
        self.slots = [_Slot(self, torch.cuda.Stream(device=self.scene.device) if slots > 1
                            else torch.cuda.current_stream(self.scene.device)) for _ in range(slots)]
        self.copy_stream = None
        self.stage_events = None
        self.plan = upscale_plan(self.width, self.height, self.out_w, self.out_h, self.scene.device)
        # the slots as the batched C entry point sees them (splat_render_views)
        self._cslots = (_lib.SlotT * self.nslots)()
        for k, slot in enumerate(self.slots):
            cs = self._cslots[k]
            cs.workspace, cs.ws_bytes, cs.pair_capacity = _lib.ptr(slot.frame.ws), slot.frame.nbytes, slot.frame.capacity
            cs.image = slot.gimg
            cs.stream = _lib.stream_ptr(slot.stream)

    # ---- capacity -------------------------------------------------------------------------
    def calibrate(self, views, margin: float = 1.05) -> int:
        """Max (tile, splat) pair count over `views` (untimed; one small sync)."""
        lib, ds = _lib.load(), self.scene
        frame = Frame(ds.n, self.width, self.height, 1, ds.device)
        st = _lib.stream_ptr()
        totals = torch.zeros(len(views), dtype=torch.int64, device=ds.device)
        for i, v in enumerate(views):
            cv = make_view(ds, self.width, self.height, v)
            _lib.check(lib.splat_prepare_view(_lib.ptr(ds.const), ds.n, cv, self.width, self.height,
                                              _lib.ptr(frame.ws), frame.nbytes, frame.capacity, st))
            _lib.check(lib.splat_bin_tiles(ds.n, self.width, self.height, _lib.ptr(frame.ws), frame.nbytes,
                                           frame.capacity, BIN_COUNT_ONLY, st))
            totals[i] = frame.counters()[0].to(torch.int64)
        return int(int(totals.max()) * margin) + 4096

    # ---- rendering ------------------------------------------------------------------------
    def enable_stage_timing(self, enabled: bool = True):
        """Record CUDA events around every stage (single-slot pipelines only)."""
        self.stage_events = [] if enabled else None

    def render(self, views, host_out=None, keep=False, out=None):
        """Launch every view; returns the list of device outputs if keep (else None).

        host_out: optional list of pinned host tensors (ring); frame i is copied
        into host_out[i % len(host_out)] on a side stream, overlapped with rendering.
        out: optional (V, Ho, Wo, 3) float32 device tensor; view i is upscaled
        straight into out[i] (the batched layout, no extra copy).
        """
        lib, ds = self.lib, self.scene
        kept = [] if keep else None
        if out is not None:
            if not torch.is_tensor(out) or out.dim() != 4 or out.shape[0] < len(views):
                raise DimensionError("out must be a (V, Ho, Wo, 3) tensor with V >= len(views)")
            for i in range(len(views)):
                check_output(out[i], self.out_w, self.out_h, ds.device)
        if host_out is not None and self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream(device=ds.device)
        # every slot (and the copy stream) starts after the work the caller queued so far on
        # its stream: the scene upload / prepare, the Frame counter zeroing, the upscale plan
        self.fork()
        if self.BATCHED and host_out is None and self.stage_events is None and len(views):
            return self._render_batched(views, keep, out)
        for i, v in enumerate(views):
            slot = self.slots[i % self.nslots]
            cv = make_view(ds, self.width, self.height, v)
            st = _lib.stream_ptr(slot.stream)
            k = slot.flip
            slot.flip ^= 1
            if out is not None:
                dst = out[i]
            elif keep:
                dst = torch.empty((self.out_h, self.out_w, 3), dtype=torch.float32, device=ds.device)
            else:
                dst = slot.out[k]
            if slot.copied[k] is not None:
                slot.stream.wait_event(slot.copied[k])
            ev = self.stage_events
            if ev is not None:
                marks = [torch.cuda.Event(enable_timing=True) for _ in range(len(STAGES) + 1)]
                marks[0].record(slot.stream)
            fw = slot.frame
            _lib.check(lib.splat_prepare_view(_lib.ptr(ds.const), ds.n, cv, self.width, self.height,
                                              _lib.ptr(fw.ws), fw.nbytes, fw.capacity, st))
            if ev is not None:
                marks[1].record(slot.stream)
            _lib.check(lib.splat_bin_tiles(ds.n, self.width, self.height, _lib.ptr(fw.ws), fw.nbytes,
                                           fw.capacity, 0, st))
            if ev is not None:
                marks[2].record(slot.stream)
            if ev is None:   # raster kernel + exact fix-up in one call
                _lib.check(lib.splat_rasterize(_lib.ptr(ds.const), ds.n, cv, self.width, self.height, 0,
                                               slot.gimg, _lib.ptr(fw.ws), fw.nbytes, fw.capacity, st))
            else:            # stage timing: the two kernels separately (different rooflines)
                _lib.check(lib.splat_rasterize(_lib.ptr(ds.const), ds.n, cv, self.width, self.height,
                                               DEFER_FIXUP, slot.gimg, _lib.ptr(fw.ws), fw.nbytes, fw.capacity,
                                               st))
                marks[3].record(slot.stream)
                _lib.check(lib.splat_fixup(_lib.ptr(ds.const), ds.n, cv, self.width, self.height, 0, slot.gimg,
                                           _lib.ptr(fw.ws), fw.nbytes, fw.capacity, st))
                marks[4].record(slot.stream)
            _lib.check(lib.splat_upscale_forward(_lib.ptr(slot.img.planes), self.width, self.height,
                                                 _lib.ptr(dst), self.out_w, self.out_h, 1,
                                                 _lib.ptr(self.plan), st))
            if ev is not None:
                marks[5].record(slot.stream)
                ev.append(marks)
            if host_out is not None:
                done = torch.cuda.Event()
                done.record(slot.stream)
                self.copy_stream.wait_event(done)
                with torch.cuda.stream(self.copy_stream):
                    host_out[i % len(host_out)].copy_(dst, non_blocking=True)
                cp = torch.cuda.Event()
                cp.record(self.copy_stream)
                slot.copied[k] = cp
            if keep:
                kept.append(dst)
        return kept

    def _render_batched(self, views, keep, out):
        """The whole batch through splat_render_views: one C call enqueues every view's
        prepare -> bin -> raster -> fix-up -> upscale chain on its slot's stream."""
        lib, ds = self.lib, self.scene
        n = len(views)
        cviews = (_lib.ViewT * n)(*[make_view(ds, self.width, self.height, v) for v in views])
        dsts = []
        for i in range(n):
            slot = self.slots[i % self.nslots]
            if out is not None:
                dsts.append(out[i])
            elif keep:
                dsts.append(torch.empty((self.out_h, self.out_w, 3), dtype=torch.float32, device=ds.device))
            else:
                dsts.append(slot.out[slot.flip])
                slot.flip ^= 1
        ptrs = (ctypes.c_void_p * n)(*[d.data_ptr() for d in dsts])
        _lib.check(lib.splat_render_views(_lib.ptr(ds.const), ds.n, cviews, n, self.width, self.height,
                                          self._cslots, self.nslots, ptrs, self.out_w, self.out_h, 1,
                                          _lib.ptr(self.plan)))
        return dsts if keep else None

    def join(self, stream=None):
        """Make `stream` (default: current) wait for all slot streams and copies."""
        s = stream or torch.cuda.current_stream(self.scene.device)
        for slot in self.slots:
            if slot.stream is not s:
                e = torch.cuda.Event()
                e.record(slot.stream)
                s.wait_event(e)
        if self.copy_stream is not None:
            e = torch.cuda.Event()
            e.record(self.copy_stream)
            s.wait_event(e)

    def fork(self, stream=None):
        """Make all slot streams wait for `stream` (default: current)."""
        s = stream or torch.cuda.current_stream(self.scene.device)
        e = torch.cuda.Event()
        e.record(s)
        for slot in self.slots:
            if slot.stream is not s:
                slot.stream.wait_event(e)
        if self.copy_stream is not None:
            self.copy_stream.wait_event(e)

    def check(self):
        """Raise if any view overflowed its pair buffer (syncs)."""
        for slot in self.slots:
            c = slot.frame.counters()
            if int(c[4].item()):
                raise RuntimeError("tile-pair capacity overflow; re-run with a larger capacity")

    def stage_times_ms(self):
        """Mean per-stage milliseconds over recorded views (call after synchronize)."""
        if not self.stage_events:
            return {}
        tot = [0.0] * len(STAGES)
        for marks in self.stage_events:
            for j in range(len(STAGES)):
                tot[j] += marks[j].elapsed_time(marks[j + 1])
        n = len(self.stage_events)
        return {s: t / n for s, t in zip(STAGES, tot)}


def render_upscale_views(scene, width: int, height: int, views, *, factor: float = 4.0, out_size=None,
                         slots: int = 4) -> torch.Tensor:
    """Batched variant of ``upscale_spline(render_forward(scene, W, H, view=v), factor)``
    for every view: returns a (V, Ho, Wo, 3) float32 device tensor."""
    pipe = ViewPipeline(scene, width, height, factor=factor, out_size=out_size, slots=slots,
                        views_for_capacity=list(views))
    out = torch.empty((len(views), pipe.out_h, pipe.out_w, 3), dtype=torch.float32, device=pipe.scene.device)
    pipe.fork()
    pipe.render(list(views), out=out)
    pipe.join()
    pipe.check()
    return out
