"""Device-resident market: the HBM layout of DESIGN.md §3, owned by torch.

    row_ptr  int64 [n+1 (+pad)]   w       float64 [n (+pad)]   scales float64 [n]
    col      int32 [nnz (+pad)]   u       float64 [nnz (+pad)] (row max 1)
    u_orig   float64 [nnz]        (residuals are measured on the original data)
    tiles    int64 [ntiles, 4]    (r0, r1, e0, e1): rows / entries of each tile
    long_rows int32 [nlong]       rows longer than 1024 entries
    med_rows int32 [nmed]         tile rows longer than 128 entries (warp per row)
    bperm    int32 [nnz]          tile-blocked transpose schedule: per block of
    bptr     int32 [(nblk+1)m+1]  4 x prim_grid tiles, per good, ascending rows
                                  (block nblk empty)
    tperm / tptr                  the reference's global schedule (sparse.py:
                                  130-145), only for the k-section drop-in
(pad) = 16 readable elements past the end for the TMA bulk copies.

Built once per instance (or per row shard); every later call only passes the
`mq_market` struct of raw pointers to the native library.
"""

import math
import os
import ctypes
import warnings

import numpy as np
import torch

from . import _native as nat


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _padded(src, dtype, device):
    """Copy of `src` with nat.PAD extra (zero) elements; returns (buffer, view)."""
    n = int(src.numel()) if isinstance(src, torch.Tensor) else len(src)
    buf = torch.zeros(n + nat.PAD, dtype=dtype, device=device)
    if n:
        if isinstance(src, torch.Tensor):
            buf[:n].copy_(src)
        else:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                buf[:n].copy_(torch.from_numpy(np.ascontiguousarray(src)))
    return buf, buf[:n]


def build_tiles(row_ptr, tile_entries=nat.TILE_ENTRIES, long_row=nat.LONG_ROW,
                tile_rows=nat.TILE_ROWS):
    """Greedy tiles: contiguous runs of rows with <= tile_entries entries and
    <= tile_rows rows, each tile as long as the next row still fits; rows
    longer than long_row break the runs and go to a separate list.
    Returns (tiles [k,2] int64, long int32).

    Greedy packing is sequential; here it is the orbit of row 0 under
    nxt(i) = end of the tile that starts at row i, found by pointer doubling
    (log2 n gathers), so it runs on the device in milliseconds at n = 1e7."""
    dev = row_ptr.device
    n = row_ptr.numel() - 1
    lens = row_ptr[1:] - row_ptr[:-1]
    is_long = lens > long_row
    long_rows = torch.nonzero(is_long).flatten().to(torch.int32)
    if int((~is_long).sum().item()) == 0:
        return torch.zeros(0, 2, dtype=torch.int64, device=dev), long_rows
    rows = torch.arange(n, device=dev)
    # first long row at or after each row (n: none)
    nl = torch.where(is_long, rows, torch.full_like(rows, n))
    seg_end = torch.flip(torch.cummin(torch.flip(nl, [0]), 0).values, [0])
    # rows i..j-1 hold at most tile_entries entries
    j_e = torch.searchsorted(row_ptr, row_ptr[:-1] + tile_entries, right=True) - 1
    nxt = torch.minimum(torch.minimum(j_e, rows + tile_rows), seg_end)
    nxt = torch.where(is_long, rows + 1, nxt)  # a long row is stepped over
    jump = torch.cat([nxt, torch.tensor([n], dtype=nxt.dtype, device=dev)])
    starts = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(max(1, n.bit_length()) + 1):
        starts = torch.unique(torch.cat([starts, jump[starts]]))
        jump = jump[jump]
    starts = starts[starts < n]
    starts = starts[~is_long[starts]]
    tiles = torch.stack([starts, nxt[starts]], 1).contiguous()
    return tiles, long_rows


def medium_rows(row_ptr, long_rows, reg_row=nat.REG_ROW):
    """Tile rows longer than reg_row (the register capacity of a tile row
    solve), longest first: the warp-per-row kernel claims them in order.
    Returns int32 [nmed]."""
    lens = row_ptr[1:] - row_ptr[:-1]
    med = lens > reg_row
    if long_rows.numel():
        med[long_rows.to(torch.int64)] = False
    rows = torch.nonzero(med).flatten()
    if rows.numel() > 1:
        rows = rows[torch.argsort(lens[rows], descending=True, stable=True)]
    return rows.to(torch.int32).contiguous()


TILES_PER_CTA_PER_BLOCK = int(os.environ.get("MQ_TILES_PER_CTA", "4"))  # tuning override


def sm_count(device):
    return torch.cuda.get_device_properties(device).multi_processor_count


def build_blocked_schedule(row_ptr, col, m, tiles, long_rows, prim_grid,
                           tiles_per_cta=TILES_PER_CTA_PER_BLOCK, tiles_per_block=None):
    """Entry positions grouped by (block of tiles, good), ascending inside a
    good.  A block covers the entries from its first tile's start to the next
    block's (long rows between tiles included), so walking a good block by
    block visits its entries in ascending row order: the reference's
    column_sums order (np.bincount over storage order, sparse.py:200-210).
    The last block index nblk is kept (empty) for the layout.  Returns
    (bperm int32 [nnz], bptr int32 [(nblk+1)*m+1], nblk, tiles_per_block)."""
    dev = col.device
    nnz = col.numel()
    ntiles = int(tiles.shape[0])
    tpb = tiles_per_block or max(1, tiles_per_cta * max(1, prim_grid))
    nblk = -(-ntiles // tpb)
    pos = torch.arange(nnz, device=dev, dtype=torch.int64)
    if nblk:
        starts = row_ptr[tiles[::tpb, 0]].contiguous()
        blk = (torch.searchsorted(starts, pos, right=True) - 1).clamp_(min=0)
    else:
        blk = torch.zeros(nnz, dtype=torch.int64, device=dev)
    del pos
    total = (nblk + 1) * m
    if total < 2 ** 31:
        key = blk.to(torch.int32) * m + col
    else:
        key = blk * m + col.to(torch.int64)
    del blk
    _, perm = torch.sort(key, stable=True)
    bperm = torch.zeros(nnz + nat.PAD, dtype=torch.int32, device=dev)
    bperm[:nnz] = perm
    del perm
    counts = torch.bincount(key.to(torch.int64), minlength=total)
    del key
    bptr = torch.zeros(total + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=bptr[1:])
    bptr32 = torch.zeros(total + 1 + nat.PAD, dtype=torch.int32, device=dev)
    bptr32[:total + 1] = bptr
    return bperm[:nnz], bptr32[:total + 1], nblk, tpb


def fixed_point_scale(max_col_count):
    """(cs_scale, cs_xmax) of the fixed-point column sums: cs_scale = 2^k,
    2^-48 <= resolution <= 2^-24, aiming at cs_xmax ~ 1024, with
    cs_xmax * cs_scale * max_col_count = 2^62 (no u64 overflow)."""
    c = max(1, int(max_col_count))
    k = int(min(48, max(24, math.floor(62 - math.log2(c) - 10))))
    return float(2.0 ** k), float(2.0 ** (62 - k) / c)


class DeviceMarket:
    """CSR utilities + budgets on one GPU (optionally a row shard).

    row_ptr (n+1), col (nnz), u_orig (nnz, original utilities), w (n) are host
    numpy arrays or device tensors; m is the (global) number of goods;
    row_begin the global index of the first row.
    """

    def __init__(self, row_ptr, col, u_orig, w, m, device=None, row_begin=0, lib=None):
        self.lib = lib or nat.lib()
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev

        def up(a, dtype):
            # transfer first, convert on the device (a host-side int64 -> int32
            # pass over 1e9 indices costs seconds)
            if not isinstance(a, torch.Tensor):
                from .engine import to_device

                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    a = to_device(a, dev)
            return a.to(device=dev).to(dtype=dtype).contiguous()

        with torch.cuda.device(dev):
            self._rp_buf, self.row_ptr = _padded(up(row_ptr, torch.int64), torch.int64, dev)
            self.n = int(self.row_ptr.numel() - 1)
            self.m = int(m)
            self._col_buf, self.col = _padded(up(col, torch.int32), torch.int32, dev)
            self.nnz = int(self.col.numel())
            self.u_orig = up(u_orig, torch.float64)
            self._w_buf, self.w = _padded(up(w, torch.float64), torch.float64, dev)
            self.row_begin = int(row_begin)
            if int(self.row_ptr[-1].item()) != self.nnz:
                raise ValueError("row_ptr[-1] does not match nnz")
            if self.nnz >= 2 ** 31:
                raise ValueError("a shard must hold < 2^31 entries (int32 positions)")
            # normalization on device (instance.py:118-138, same IEEE division)
            self._u_buf = torch.zeros(self.nnz + nat.PAD, dtype=torch.float64, device=dev)
            self.u = self._u_buf[:self.nnz]
            self.scales = torch.empty(self.n, dtype=torch.float64, device=dev)
            nat.check(self.lib.mq_normalize_rows(self.n, nat.ptr(self.row_ptr),
                                                 nat.ptr(self.u_orig), nat.ptr(self.u),
                                                 nat.ptr(self.scales), _stream()),
                      "mq_normalize_rows")
            self.col_counts = (torch.bincount(self.col.to(torch.int64), minlength=self.m)
                               if self.nnz else torch.zeros(self.m, dtype=torch.int64,
                                                            device=dev))
            etile = int(self.lib.mq_tile_entries())
            tiles2, self.long_rows = build_tiles(self.row_ptr, etile,
                                                 min(nat.LONG_ROW, etile // 2))
            if self.long_rows.numel() > 1:  # longest first: the CTAs claim them in order
                lr = self.long_rows.to(torch.int64)
                order = torch.argsort(self.row_ptr[lr + 1] - self.row_ptr[lr], descending=True,
                                      stable=True)
                self.long_rows = self.long_rows[order].contiguous()
            self.med_rows = medium_rows(self.row_ptr, self.long_rows, int(self.lib.mq_reg_row()))
            # (r0, r1, e0, e1) per tile: the producer warp needs no dependent loads
            self.tiles = torch.cat([tiles2, self.row_ptr[tiles2]], 1).contiguous()
            self.prim_grid = int(min(max(1, self.tiles.shape[0]), sm_count(dev)))
            # the blocked schedule orders the deterministic fp64 column sums of
            # the residual checks (mq_colsum)
            self.bperm, self.bptr, self.nblk, self.tiles_per_block = build_blocked_schedule(
                self.row_ptr, self.col, self.m, tiles2, self.long_rows, self.prim_grid)
            self.max_col_count = int(self.col_counts.max().item()) if self.m else 0
            lens = self.row_ptr[1:] - self.row_ptr[:-1]
            self.max_row_len = int(lens.max().item()) if self.n else 0
        self.tperm = self.tptr = None
        self.colsum_mode = int(self.lib.mq_colsum_mode())
        self.struct = self._make_struct()

    def global_schedule(self):
        """(tperm int32, tptr int64): the reference's transpose schedule, for
        the k-section drop-in (built on first use)."""
        if self.tperm is None:
            with torch.cuda.device(self.device):
                _, perm = torch.sort(self.col, stable=True)
                self.tperm = perm.to(torch.int32)
                self.tptr = torch.zeros(self.m + 1, dtype=torch.int64, device=self.device)
                torch.cumsum(self.col_counts, 0, out=self.tptr[1:])
        return self.tperm, self.tptr

    def _make_struct(self):
        s = nat.MqMarket()
        s.n, s.m, s.nnz = self.n, self.m, self.nnz
        s.row_ptr = self.row_ptr.data_ptr()
        s.col = self.col.data_ptr()
        s.u = self.u.data_ptr()
        s.u_orig = self.u_orig.data_ptr()
        s.w = self.w.data_ptr()
        s.tiles = self.tiles.data_ptr()
        s.ntiles = int(self.tiles.shape[0])
        s.long_rows = self.long_rows.data_ptr()
        s.nlong = int(self.long_rows.numel())
        s.med_rows = self.med_rows.data_ptr()
        s.nmed = int(self.med_rows.numel())
        if s.nmed:  # med_rows is longest first
            ml = (self.row_ptr[self.med_rows.to(torch.int64) + 1]
                  - self.row_ptr[self.med_rows.to(torch.int64)])
            s.nmed_long = int((ml > nat.WS_MAX_ROW).sum().item())
        s.bperm = self.bperm.data_ptr()
        s.bptr = self.bptr.data_ptr()
        s.nblk = int(self.nblk)
        s.tiles_per_block = int(self.tiles_per_block)
        s.prim_grid = int(self.prim_grid)
        s.row_begin = self.row_begin
        s.cs_scale, s.cs_xmax = fixed_point_scale(self.max_col_count)
        return s

    @classmethod
    def from_instance(cls, inst, device=None, lib=None):
        u = inst.utilities
        return cls(u.row_offsets, u.col_indices, u.values, inst.budgets,
                   u.n_cols, device=device, lib=lib)

    def set_budgets(self, w):
        """Replace budgets in place (Arrow-Debreu outer loop)."""
        if not isinstance(w, torch.Tensor):
            w = torch.as_tensor(np.asarray(w, dtype=np.float64))
        self.w.copy_(w)

    def bytes_resident(self):
        ts = [self._rp_buf, self._col_buf, self._u_buf, self.u_orig, self._w_buf, self.scales,
              self.tiles, self.long_rows, self.med_rows, self.bperm, self.bptr]
        if self.tperm is not None:
            ts += [self.tperm, self.tptr]
        return sum(t.numel() * t.element_size() for t in ts)
