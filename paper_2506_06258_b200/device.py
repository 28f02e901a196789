"""Device-resident market: the HBM layout of DESIGN.md §3, owned by torch.

    row_ptr  int64 [n+1]    col    int32 [nnz]   u  float64 [nnz] (row max 1)
    u_orig   float64 [nnz]  w      float64 [n]   scales float64 [n]
    tptr     int64 [m+1]    tperm  int32 [nnz]   (stable column grouping)
    bin_rows int32 [n]      rows grouped by length bin for the primal kernels

Built once per instance (or per shard); every later call only passes the
`mq_market` struct of raw pointers to the native library.
"""

import numpy as np
import torch

from . import _native as nat

# upper row length of bins 0..7 of the primal kernel (bin 8 = longer rows)
BIN_EDGES = (4, 8, 16, 32, 64, 128, 256, 512)


def _stream():
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(s):
    import ctypes

    return ctypes.c_void_p(s.cuda_stream)


class DeviceMarket:
    """CSR utilities + budgets on one GPU (optionally a row shard).

    Parameters are host numpy arrays or device tensors: row_ptr (n+1),
    col (nnz), u_orig (nnz, original utilities), w (n).  m is the number of
    goods (global).  row_begin is the global index of the first row.
    """

    def __init__(self, row_ptr, col, u_orig, w, m, device=None, row_begin=0, lib=None):
        self.lib = lib or nat.lib()
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev

        def up(a, dtype):
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=dtype).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)

        with torch.cuda.device(dev):
            self.row_ptr = up(row_ptr, torch.int64)
            self.col = up(col, torch.int32)
            self.u_orig = up(u_orig, torch.float64)
            self.w = up(w, torch.float64)
            self.n = int(self.row_ptr.numel() - 1)
            self.m = int(m)
            self.nnz = int(self.col.numel())
            self.row_begin = int(row_begin)
            if int(self.row_ptr[-1].item()) != self.nnz:
                raise ValueError("row_ptr[-1] does not match nnz")
            # normalization on device (instance.py:118-138, same IEEE division)
            self.u = torch.empty_like(self.u_orig)
            self.scales = torch.empty(self.n, dtype=torch.float64, device=dev)
            nat.check(self.lib.mq_normalize_rows(self.n, nat.ptr(self.row_ptr), nat.ptr(self.u_orig),
                                                 nat.ptr(self.u), nat.ptr(self.scales), _stream()),
                      "mq_normalize_rows")
            # transpose schedule: stable sort of columns = ascending row inside
            # every column (sparse.py:130-145)
            if self.nnz:
                _, perm = torch.sort(self.col, stable=True)
                self.tperm = perm.to(torch.int32)
                del perm
                counts = torch.bincount(self.col.to(torch.int64), minlength=self.m)
            else:
                self.tperm = torch.zeros(0, dtype=torch.int32, device=dev)
                counts = torch.zeros(self.m, dtype=torch.int64, device=dev)
            self.col_counts = counts
            self.tptr = torch.zeros(self.m + 1, dtype=torch.int64, device=dev)
            torch.cumsum(counts, 0, out=self.tptr[1:])
            # row-length bins for the primal kernels
            lens = self.row_ptr[1:] - self.row_ptr[:-1]
            edges = torch.tensor(BIN_EDGES, dtype=torch.int64, device=dev)
            bins = torch.bucketize(lens, edges, right=False)
            order = torch.sort(bins, stable=True)[1]
            self.bin_rows = order.to(torch.int32)
            bc = torch.bincount(bins, minlength=len(BIN_EDGES) + 1).cpu().numpy()
            self.bin_off = np.zeros(len(BIN_EDGES) + 2, dtype=np.int64)
            self.bin_off[1:] = np.cumsum(bc)
            self.max_row_len = int(lens.max().item()) if self.n else 0
        self.struct = self._make_struct()

    def _make_struct(self):
        s = nat.MqMarket()
        s.n, s.m, s.nnz = self.n, self.m, self.nnz
        s.row_ptr = self.row_ptr.data_ptr()
        s.col = self.col.data_ptr()
        s.u = self.u.data_ptr()
        s.u_orig = self.u_orig.data_ptr()
        s.w = self.w.data_ptr()
        s.tptr = self.tptr.data_ptr()
        s.tperm = self.tperm.data_ptr()
        s.bin_rows = self.bin_rows.data_ptr()
        for k in range(nat.NBINS + 1):
            s.bin_off[k] = int(self.bin_off[k])
        s.row_begin = self.row_begin
        return s

    @classmethod
    def from_instance(cls, inst, device=None, lib=None):
        u = inst.utilities
        return cls(u.row_offsets, u.col_indices.astype(np.int32), u.values, inst.budgets,
                   u.n_cols, device=device, lib=lib)

    def set_budgets(self, w):
        """Replace budgets in place (Arrow-Debreu outer loop)."""
        self.w.copy_(torch.as_tensor(np.asarray(w, dtype=np.float64)) if not isinstance(
            w, torch.Tensor) else w)

    def bytes_resident(self):
        ts = (self.row_ptr, self.col, self.u, self.u_orig, self.w, self.scales, self.tptr,
              self.tperm, self.bin_rows)
        return sum(t.numel() * t.element_size() for t in ts)
