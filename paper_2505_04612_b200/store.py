"""Device-resident data layouts of the hot path and their (bit-exact) builders.

* :class:`PointPairStore` -- the per-point data of a list of ``EpipolarPair``
  (ref/epipolar.py:19-36) re-laid out as a structure of arrays in HBM: fp32
  ``(x, y)`` columns for each image side, a 1-bit active mask, image pairs
  sorted by ``(i, j)`` (stable, so duplicates keep caller order), each pair
  starting on a 16-slot boundary (SLOT_ALIGN).  ``terms`` (72 B/point in the reference) is
  never stored: the kernels rebuild ``flatten(x2 x1^T)`` in registers.
* :class:`PairGraph` -- image-pair -> dense-image / camera indices plus the
  incidence lists that make per-image and per-camera gradient sums
  deterministic gathers (ref/epipolar.py:163-169 remap, :219-224 scatter).
* :class:`DirGraphDevice` -- ``DirectionGraph`` (ref/translation.py:104-109)
  plus its node incidence list.

All index bookkeeping is integer numpy (exact); the float payload is uploaded
once and stays on the device.
"""

import ctypes

import numpy as np
import torch

from . import _native as N

CHUNK = 8192          # slots per work item (multiple of 128)
SLOT_ALIGN = 16       # pair start alignment (slots): whole 16-slot blocks for the hot kernel
CAM_CHUNK = 1024      # incidences per camera-reduction chunk (256 and 4096 measured slower)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(t):
    return t.data_ptr() if t is not None else None


def _dev(a, device):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device, non_blocking=False)


def pair_order(i, j):
    """Stable (i, j) order of image pairs (ref/tracks.py:104 sorts this way)."""
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    return np.lexsort((j, i)).astype(np.int64)


def slot_layout(lengths, chunk=CHUNK):
    """SLOT_ALIGN-aligned slot offsets and work items for per-pair point counts.

    Returns (pair_off [P+1] int64, n_slots, pair_item_off [P+1] int32,
    item_pair [n_items] int32).
    """
    lengths = np.asarray(lengths, dtype=np.int64)
    P = len(lengths)
    padded = (lengths + SLOT_ALIGN - 1) // SLOT_ALIGN * SLOT_ALIGN
    pair_off = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(padded, out=pair_off[1:])
    n_slots = int((pair_off[-1] + 127) // 128 * 128)
    n_slots = max(n_slots, 128)
    items = np.maximum(1, (lengths + chunk - 1) // chunk)
    pair_item_off = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(items, out=pair_item_off[1:])
    item_pair = np.repeat(np.arange(P, dtype=np.int64), items)
    if pair_item_off[-1] >= 2**31:
        raise ValueError("too many work items")
    return pair_off, n_slots, _i32(pair_item_off), _i32(item_pair)


class PointPairStore:
    """SoA point-pair store on one device.

    ``order[k]`` is the caller index of the k-th stored pair; ``rank`` is its
    inverse.  The host computes only the O(pairs) layout; the O(points) work
    -- scatter into 16-slot aligned pairs, fp64 -> fp32, sanitising, mask
    packing -- is ``fm_store_build`` on the device, and the per-point maps
    back to caller order are ``fm_store_gather_*`` (no host point_slot array).
    """

    def __init__(self, x1, x2, lengths, pair_i, pair_j, active=None, device=None,
                 chunk=CHUNK, order=None, sanitize=False, fp64=False):
        """x1, x2: (Z, 2) or (Z, 3) float arrays of all points, pairs in caller
        order; lengths: points per pair (caller order).

        sanitize=True zeroes the coordinates of non-finite points and clears
        their active bit.  The IRLS moment passes need finite coordinates on
        every slot; for irls_refine this is exactly the reference's behaviour
        (a non-finite residual fails ``res <= th`` in the first prune,
        ref/epipolar.py:283).  API stores (current_residuals) keep NaNs.

        fp64=True keeps the caller's fp64 (x, y, z) coordinates ([n_slots][3],
        48 B per point pair) instead of the fp32 hot-store columns: the API
        functions (precompute_weights, current_residuals, epipolar_loss) then
        compute on exactly the reference's inputs.  irls_refine uses the fp32
        hot store (north star: fp32 storage, 1e-4 tolerance)."""
        device = device or N.require_cuda()
        lengths = np.asarray(lengths, dtype=np.int64)
        P = len(lengths)
        self.device = device
        self.n_pairs = P
        self.chunk = chunk
        if order is None:
            order = pair_order(pair_i, pair_j)
        self.order = np.asarray(order, dtype=np.int64)
        self.rank = np.empty(P, dtype=np.int64)
        self.rank[self.order] = np.arange(P)
        self.len_caller = lengths
        s_len = lengths[self.order]
        pair_off, n_slots, pair_item_off, item_pair = slot_layout(s_len, chunk)
        self.pair_off = pair_off
        self.n_slots = n_slots
        self.n_items = len(item_pair)
        self.n_points = int(lengths.sum())
        self.caller_start = np.zeros(P + 1, dtype=np.int64)
        np.cumsum(lengths, out=self.caller_start[1:])
        self.sanitized = bool(sanitize)
        self.fp64 = bool(fp64)

        x1 = np.asarray(x1, dtype=np.float64)
        x2 = np.asarray(x2, dtype=np.float64)
        dim = x1.shape[1] if x1.ndim == 2 and len(x1) else 2
        if self.n_points:
            x1d = _dev(np.ascontiguousarray(x1), device)
            x2d = _dev(np.ascontiguousarray(x2), device)
            act = None if active is None else _dev(np.asarray(active, dtype=np.uint8), device)
        else:  # pairs without points: nothing is read
            x1d = x2d = torch.zeros((1, dim), dtype=torch.float64, device=device)
            act = None
        # z != 1 anywhere needs the homogeneous columns; decided on the device
        # (a strided host scan of the z column cost ~30 ms per side at C2)
        homog = (not fp64 and dim == 3 and self.n_points > 0
                 and not bool(((x1d[:, 2] == 1.0).all() & (x2d[:, 2] == 1.0).all()).item()))
        self.homogeneous = bool(homog)
        self.x1d = self.x2d = self.x1 = self.x2 = self.x1z = self.x2z = None
        if fp64:
            self.x1d = torch.empty((n_slots, 3), dtype=torch.float64, device=device)
            self.x2d = torch.empty((n_slots, 3), dtype=torch.float64, device=device)
        else:
            self.x1 = torch.empty((n_slots, 2), dtype=torch.float32, device=device)
            self.x2 = torch.empty((n_slots, 2), dtype=torch.float32, device=device)
            if homog:
                self.x1z = torch.empty(n_slots, dtype=torch.float32, device=device)
                self.x2z = torch.empty(n_slots, dtype=torch.float32, device=device)
        self.active = torch.empty(n_slots // 32, dtype=torch.int32, device=device)
        self.pair_off_d = _dev(pair_off, device)
        self.pair_len_d = _dev(_i32(s_len), device)
        self.pair_item_off_d = _dev(pair_item_off, device)
        self.item_pair_d = _dev(item_pair, device)
        self.caller_start_d = _dev(self.caller_start, device)
        self.rank_d = _dev(self.rank, device)
        self._struct = None
        N.check(N.lib().fm_store_build(ctypes.byref(self.struct()), N.ptr(x1d), N.ptr(x2d), dim,
                                       N.ptr(act), N.ptr(self.caller_start_d), N.ptr(self.rank_d),
                                       int(sanitize), N.stream_handle()))
        del x1d, x2d, act

    # ---------------------------------------------------------------- ctypes
    def struct(self):
        if self._struct is None:
            self._struct = N.PointStore(
                n_pairs=self.n_pairs, n_slots=self.n_slots, n_items=self.n_items,
                chunk=self.chunk,
                pair_off=self.pair_off_d.data_ptr(), pair_len=self.pair_len_d.data_ptr(),
                pair_item_off=self.pair_item_off_d.data_ptr(),
                item_pair=self.item_pair_d.data_ptr(),
                x1=_ptr(self.x1), x2=_ptr(self.x2), x1z=_ptr(self.x1z), x2z=_ptr(self.x2z),
                active=self.active.data_ptr(), item_desc=None, slot_align=SLOT_ALIGN,
                x1d=_ptr(getattr(self, "x1d", None)), x2d=_ptr(getattr(self, "x2d", None)))
            self.item_desc_d = torch.empty((max(self.n_items, 1), 4), dtype=torch.int32,
                                           device=self.device)
            self._struct.item_desc = self.item_desc_d.data_ptr()
            N.check(N.lib().fm_point_store_describe(ctypes.byref(self._struct), N.stream_handle()))
        return self._struct

    def scratch(self):
        """Pass scratch (zeroed: fm_point_pass keeps its totals ticket there)."""
        nbytes = N.lib().fm_point_pass_scratch_bytes(ctypes.byref(self.struct()))
        return torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=self.device)

    # ----------------------------------------------- caller <-> slot order maps
    def _caller_maps(self):
        if getattr(self, "caller_start_d", None) is None:
            self.caller_start_d = _dev(self.caller_start, self.device)
            self.rank_d = _dev(self.rank, self.device)
        return self.caller_start_d, self.rank_d

    def gather_slots(self, slot_values):
        """Per-slot fp64 values -> caller point order (device tensor [Z])."""
        cs, rk = self._caller_maps()
        out = torch.empty(max(self.n_points, 1), dtype=torch.float64, device=self.device)
        N.check(N.lib().fm_store_gather_slots(ctypes.byref(self.struct()), N.ptr(cs), N.ptr(rk),
                                              N.ptr(slot_values), N.ptr(out), N.stream_handle()))
        return out[:self.n_points]

    def scatter_slots(self, caller_values):
        """Caller-ordered fp64 values [Z] -> a per-slot device tensor (0 on padding)."""
        cs, rk = self._caller_maps()
        src = torch.as_tensor(np.ascontiguousarray(caller_values, dtype=np.float64), device=self.device)
        out = torch.zeros(self.n_slots, dtype=torch.float64, device=self.device)
        N.check(N.lib().fm_store_scatter_slots(ctypes.byref(self.struct()), N.ptr(cs), N.ptr(rk),
                                               N.ptr(src), N.ptr(out), N.stream_handle()))
        return out

    # ------------------------------------------------------------- masks
    def active_bits(self):
        """Active flag of every slot (device bool tensor)."""
        words = self.active.view(torch.int32)
        shifts = torch.arange(32, device=self.device, dtype=torch.int32)
        return ((words.unsqueeze(1) >> shifts) & 1).reshape(-1).bool()

    def caller_masks(self):
        """Active mask of every caller point, host bool array (caller order)."""
        cs, rk = self._caller_maps()
        out = torch.empty(max(self.n_points, 1), dtype=torch.uint8, device=self.device)
        N.check(N.lib().fm_store_gather_mask(ctypes.byref(self.struct()), N.ptr(cs), N.ptr(rk),
                                             N.ptr(out), N.stream_handle()))
        return out[:self.n_points].cpu().numpy().astype(bool)

    def write_back(self, pairs):
        """In-place update of each pair's ``active`` array (ref/epipolar.py:283)."""
        masks = self.caller_masks()
        for k, p in enumerate(pairs):
            seg = masks[self.caller_start[k]:self.caller_start[k + 1]]
            if isinstance(p.active, np.ndarray) and p.active.dtype == bool and p.active.shape == seg.shape:
                p.active[...] = seg
            else:
                p.active = seg.copy()

    def to_stored(self, per_pair_caller):
        return np.asarray(per_pair_caller)[self.order]

    @classmethod
    def from_device(cls, x1, x2, lengths, device, chunk=CHUNK):
        """Build from device tensors x1, x2 (Z, 2) float32 whose pairs are
        already in (i, j) order with ``lengths`` points each (all active)."""
        self = cls.__new__(cls)
        lengths = np.asarray(lengths, dtype=np.int64)
        P = len(lengths)
        self.device = device
        self.n_pairs = P
        self.chunk = chunk
        self.order = np.arange(P, dtype=np.int64)
        self.rank = self.order.copy()
        self.len_caller = lengths
        pair_off, n_slots, pair_item_off, item_pair = slot_layout(lengths, chunk)
        self.pair_off = pair_off
        self.n_slots = n_slots
        self.n_items = len(item_pair)
        self.n_points = int(lengths.sum())
        self.caller_start = np.zeros(P + 1, dtype=np.int64)
        np.cumsum(lengths, out=self.caller_start[1:])
        lens_d = torch.as_tensor(lengths, device=device)
        seg = torch.repeat_interleave(torch.arange(P, device=device), lens_d)
        start_d = torch.as_tensor(self.caller_start[:-1], device=device)
        off_d = torch.as_tensor(pair_off[:-1], device=device)
        slot = off_d[seg] + (torch.arange(self.n_points, device=device) - start_d[seg])
        del seg
        self.point_slot_d = slot
        self.x1 = torch.zeros((n_slots, 2), dtype=torch.float32, device=device)
        self.x2 = torch.zeros((n_slots, 2), dtype=torch.float32, device=device)
        self.x1[slot] = x1.to(torch.float32)
        self.x2[slot] = x2.to(torch.float32)
        self.x1z = self.x2z = self.x1d = self.x2d = None
        self.homogeneous = False
        self.fp64 = False
        self.sanitized = True  # device-generated coordinates are finite
        self.active = torch.zeros(n_slots // 32, dtype=torch.int32, device=device)
        self.pair_off_d = _dev(pair_off, device)
        self.pair_len_d = _dev(_i32(lengths), device)
        self.pair_item_off_d = _dev(pair_item_off, device)
        self.item_pair_d = _dev(item_pair, device)
        self.caller_start_d = None
        self._struct = None
        self.reset_active()
        return self

    def reset_active(self):
        """Mark every real point active again (benchmark repetitions)."""
        slot = getattr(self, "point_slot_d", None)
        if slot is None:
            slot = self.gather_slots(torch.arange(self.n_slots, device=self.device,
                                                  dtype=torch.float64)).long()
        bits = torch.zeros(self.n_slots, dtype=torch.int64, device=self.device)
        bits[slot] = 1
        w = (bits.view(-1, 32) << torch.arange(32, device=self.device, dtype=torch.int64)).sum(1)
        self.active.copy_(torch.where(w >= 2**31, w - 2**32, w).to(torch.int32))

    @classmethod
    def from_pairs(cls, pairs, device=None, chunk=CHUNK, all_active=False, sanitize=False,
                   fp64=False):
        """Build from EpipolarPair-like objects (reference or ours)."""
        lengths = np.fromiter((len(p.x1) for p in pairs), dtype=np.int64, count=len(pairs))
        if len(pairs):
            rows = int(lengths.sum())
            x1 = _stack_rows([p.x1 for p in pairs], np.float64, 3, "x1", rows)
            x2 = _stack_rows([p.x2 for p in pairs], np.float64, 3, "x2", rows)
            act = None if all_active else _stack_rows([p.active for p in pairs], bool, None, "act", rows)
        else:
            x1 = np.zeros((0, 3))
            x2 = np.zeros((0, 3))
            act = None
        i = np.fromiter((p.i for p in pairs), dtype=np.int64, count=len(pairs))
        j = np.fromiter((p.j for p in pairs), dtype=np.int64, count=len(pairs))
        return cls(x1, x2, lengths, i, j, active=act, device=device, chunk=chunk, sanitize=sanitize,
                   fp64=fp64)


# Host staging of the API store build: page-locked, reused across calls
# (grow-only, per column), so the concatenation writes warm pages and the
# upload is a DMA at full PCIe speed instead of a staged pageable copy.
# Calls are stream-ordered and synchronised at their end (irls_refine and
# the API functions read results back), so a buffer is free again when the
# next call fills it.  Columns above the cap use ordinary memory.
_STAGE = {}
_STAGE_CAP = 1 << 30  # bytes per column


def release_staging():
    """Free the page-locked staging buffers of the API store build (they
    are kept between calls; the next call allocates them again)."""
    _STAGE.clear()


def _staging(name, n, dtype):
    """A page-locked numpy array of n `dtype` values (a view of a cached
    pinned buffer), or None when it would exceed the cap or pinning fails."""
    nbytes = int(n) * np.dtype(dtype).itemsize
    if nbytes == 0 or nbytes > _STAGE_CAP or not torch.cuda.is_available():
        return None
    buf = _STAGE.get(name)
    if buf is None or buf.numel() < nbytes:
        try:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        except RuntimeError:
            return None
        _STAGE[name] = buf
    return buf.numpy()[:nbytes].view(dtype)


def _stack_rows(arrays, dtype, width, stage=None, rows=None):
    """np.concatenate of per-pair arrays as (-1, width) (or flat) `dtype`
    rows: one concatenate when every array already has that dtype and shape
    (the pipeline's EpipolarPair), else a per-array conversion.  stage: name
    of a pinned staging buffer to concatenate into; rows: the row count when
    the caller knows it (then the common case concatenates straight into the
    staging buffer, numpy checking shapes and casts, with no per-array scan)."""
    if rows is not None and stage:
        out = _staging(stage, rows * (width or 1), dtype)
        if out is not None:
            out = out.reshape((rows,) if width is None else (rows, width))
            try:
                return np.concatenate(arrays, out=out, casting="safe")
            except (ValueError, TypeError):
                pass  # ragged widths / unsafe casts: the checked path below

    def ok(a):
        return (isinstance(a, np.ndarray) and a.dtype == dtype
                and (a.ndim == 1 if width is None else (a.ndim == 2 and a.shape[1] == width)))
    if not all(ok(a) for a in arrays):
        shape = (-1,) if width is None else (-1, width)
        arrays = [np.asarray(a, dtype=dtype).reshape(shape) for a in arrays]
    rows = sum(len(a) for a in arrays)
    out = _staging(stage, rows * (width or 1), dtype) if stage else None
    if out is None:
        return np.concatenate(arrays)
    out = out.reshape((rows,) if width is None else (rows, width))
    return np.concatenate(arrays, out=out)


def csr(keys, n_keys, payload):
    """Stable CSR of payload grouped by key (keys in [0, n_keys))."""
    keys = np.asarray(keys, dtype=np.int64)
    order = np.lexsort((np.asarray(payload, dtype=np.int64), keys))
    off = np.zeros(n_keys + 1, dtype=np.int64)
    np.cumsum(np.bincount(keys, minlength=n_keys), out=off[1:])
    return _i32(off), _i32(np.asarray(payload, dtype=np.int64)[order])


class PairGraph:
    """Image-pair graph of the adjustment on one device (pairs in store order)."""

    def __init__(self, idx_i, idx_j, cam_i, cam_j, n_images, n_cameras, refine_focal,
                 device=None):
        device = device or N.require_cuda()
        self.device = device
        idx_i = np.asarray(idx_i, dtype=np.int64)
        idx_j = np.asarray(idx_j, dtype=np.int64)
        cam_i = np.asarray(cam_i, dtype=np.int64)
        cam_j = np.asarray(cam_j, dtype=np.int64)
        P = len(idx_i)
        self.n_pairs = P
        self.n_images = int(n_images)
        self.n_cameras = int(n_cameras)
        self.refine_focal = bool(refine_focal)
        if self.refine_focal and P and (min(cam_i.min(), cam_j.min()) < 0 or
                                        max(cam_i.max(), cam_j.max()) >= n_cameras):
            raise IndexError("camera id out of range of log_focal")
        inc = np.concatenate([np.arange(P) * 2, np.arange(P) * 2 + 1])
        self.img_off, self.img_inc = csr(np.concatenate([idx_i, idx_j]), self.n_images, inc)
        if self.refine_focal:
            self.cam_off, self.cam_inc = csr(np.concatenate([cam_i, cam_j]), self.n_cameras, inc)
            lo, cam, coff = [], [], [0]
            for c in range(self.n_cameras):
                a, b = int(self.cam_off[c]), int(self.cam_off[c + 1])
                for s in range(a, b, CAM_CHUNK):
                    lo.append(s)
                    cam.append(c)
                coff.append(len(lo))
            lo.append(int(self.cam_off[-1]))
            self.cam_chunk_lo = _i32(lo)
            self.cam_chunk_cam = _i32(cam if cam else [0])
            self.cam_chunk_off = _i32(coff)
        else:
            self.cam_off = _i32(np.zeros(max(self.n_cameras, 0) + 1))
            self.cam_inc = _i32([0])
            self.cam_chunk_lo = _i32([0])
            self.cam_chunk_cam = _i32([0])
            self.cam_chunk_off = _i32(np.zeros(max(self.n_cameras, 0) + 1))
        self.n_cam_chunks = len(self.cam_chunk_lo) - 1
        host = {"pair_i": _i32(idx_i), "pair_j": _i32(idx_j), "pair_ci": _i32(cam_i),
                "pair_cj": _i32(cam_j), "img_off": self.img_off, "img_inc": self.img_inc,
                "cam_off": self.cam_off, "cam_inc": self.cam_inc,
                "cam_chunk_lo": self.cam_chunk_lo, "cam_chunk_cam": self.cam_chunk_cam,
                "cam_chunk_off": self.cam_chunk_off}
        self.t = {k: _dev(v if len(v) else _i32([0]), device) for k, v in host.items()}
        self._struct = None
        self.n_params = 9 * self.n_images + (self.n_cameras if self.refine_focal else 0)

    def struct(self):
        if self._struct is None:
            t = self.t
            self._struct = N.PairGraph(
                n_images=self.n_images, n_cameras=self.n_cameras,
                refine_focal=int(self.refine_focal), n_cam_chunks=self.n_cam_chunks,
                n_pairs=self.n_pairs,
                **{k: t[k].data_ptr() for k in ("pair_i", "pair_j", "pair_ci", "pair_cj",
                                                 "img_off", "img_inc", "cam_off", "cam_inc",
                                                 "cam_chunk_lo", "cam_chunk_cam",
                                                 "cam_chunk_off")})
        return self._struct

    def scratch(self):
        nbytes = N.lib().fm_epi_scratch_bytes(ctypes.byref(self.struct()))
        return torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)


class DirGraphDevice:
    """DirectionGraph on one device with its node incidence list."""

    def __init__(self, graph, device=None):
        device = device or N.require_cuda()
        self.device = device
        ei = np.asarray(graph.edges_i, dtype=np.int64)
        ej = np.asarray(graph.edges_j, dtype=np.int64)
        m = len(ei)
        self.n = int(graph.n)
        self.m = m
        if m and (min(ei.min(), ej.min()) < 0 or max(ei.max(), ej.max()) >= self.n):
            raise IndexError("edge endpoint out of range")
        # per node: the edges where it is j (by edge id), then those where it
        # is i -- the order of the reference's np.add.at scatter
        # (ref/translation.py:123-124), which the kernels fold in
        edge = np.concatenate([np.arange(m), np.arange(m)])
        side = np.concatenate([np.zeros(m, np.int64), np.ones(m, np.int64)])
        node = np.concatenate([ei, ej])
        order = np.lexsort((edge, 1 - side, node))
        self.node_off = np.zeros(self.n + 1, dtype=np.int32)
        np.cumsum(np.bincount(node, minlength=self.n), out=self.node_off[1:])
        self.node_inc = _i32((edge * 2 + side)[order])
        self.ei = _dev(_i32(ei), device)
        self.ej = _dev(_i32(ej), device)
        self.dirs = _dev(np.asarray(graph.directions, dtype=np.float64).reshape(m, 3), device)
        self.off_d = _dev(self.node_off, device)
        self.inc_d = _dev(self.node_inc, device)
        self._struct = N.DirGraph(n_nodes=self.n, n_edges=m, edge_i=self.ei.data_ptr(),
                                  edge_j=self.ej.data_ptr(), dirs=self.dirs.data_ptr(),
                                  node_off=self.off_d.data_ptr(), node_inc=self.inc_d.data_ptr())

    def struct(self):
        return self._struct

    def scratch(self, runs):
        """Scratch of a B-run call, kept per B: fm_tr_align's captured CUDA
        graphs are keyed on the scratch pointers, so reusing it replays them
        (calls on one graph object are stream-ordered, not concurrent)."""
        cache = self.__dict__.setdefault("_scratch", {})
        if runs not in cache:
            nbytes = N.lib().fm_tr_scratch_bytes(self.n, self.m, runs)
            cache[runs] = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        return cache[runs]

    def flag(self):
        """The device error word of this graph's descents (zeroed per call)."""
        if "_flag" not in self.__dict__:
            self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._flag.zero_()
        return self._flag
