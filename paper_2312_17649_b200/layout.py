"""Packed variable-length token layout and its device-side index (K1).

The reference batches equal-length sequences sharing ONE partition
(R/encoder.py:461-468, R/bench.py:101-103).  Here a batch is packed:
sequence j occupies token rows [cu_seqlens[j], cu_seqlens[j+1]) and is split
into the cls / query / doc groups of SubsequencePartition (R/encoder.py:58-94):
cls = 1 row, query = qgroup_len[j] rows (query tokens + [SEP]), doc = the rest
(doc tokens + final [SEP]).  ``sc_index_build`` derives every per-token and
per-tile index on the device from (cu_seqlens, qgroup_len).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

DEFAULT_TILE_ROWS = 64


class LayoutError(ValueError):
    pass


def to_device(a: np.ndarray, device) -> torch.Tensor:
    """Host array -> device tensor without a host/device sync: staged through a pinned
    buffer (torch's caching host allocator keeps it alive until the copy has run), so
    the host can pack the next batch while the GPU still works on this one."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if torch.device(device).type != "cuda":
        return t.to(device)
    return t.pin_memory().to(device, non_blocking=True)


class PackedLayout:
    """Device index of a packed batch; reusable across all encoder layers."""

    def __init__(self, cu_host: np.ndarray, qlen_host: np.ndarray, device, tile_rows: int,
                 qds_every: int = 0, qds_positions=None):
        self.cu_host = np.ascontiguousarray(cu_host, dtype=np.int32)
        self.qlen_host = np.ascontiguousarray(qlen_host, dtype=np.int32)
        self.nseq = int(self.qlen_host.shape[0])
        self.total_tokens = int(self.cu_host[-1])
        self.tile_rows = int(tile_rows)
        self.device = torch.device(device)
        seq_lens = np.diff(self.cu_host)
        self.group_lens_host = np.stack(
            [np.ones(self.nseq, np.int64), self.qlen_host.astype(np.int64),
             seq_lens.astype(np.int64) - 1 - self.qlen_host], axis=1)
        self.qds_every = int(qds_every) if qds_every else 0
        dev = self.device
        T = self.total_tokens
        self.cu_seqlens = to_device(self.cu_host, dev)
        self.qgroup_len = to_device(self.qlen_host, dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.tok_seq = torch.empty(T, **i32)
        self.tok_group = torch.empty(T, **i32)
        self.tok_rel = torch.empty(T, **i32)
        self.tok_pos = torch.empty(T, **i32)
        self.cls_rows = to_device(self.cu_host[:-1].astype(np.int64), dev)  # each sequence's [CLS] row
        self.ident_cu = torch.arange(self.nseq + 1, **i32)  # row j = sequence j (per-sequence [CLS] arrays)
        self.seq_tile_base = torch.empty(self.nseq + 1, **i32)
        self.seq_head_base = torch.empty(self.nseq + 1, **i32)
        self.max_qgroup_len = int(self.qlen_host.max())
        # doc tiles of tile_rows rows over all sequences (host copy of seq_tile_base[nseq])
        self.n_tiles = int(((self.group_lens_host[:, 2] + self.tile_rows - 1) // self.tile_rows).sum())
        self.tok_flags = self.glob_cu = self.glob_pos = None
        if self.qds_every or qds_positions is not None:
            self.tok_flags = torch.zeros(T, dtype=torch.uint8, device=dev)
            self.glob_cu = torch.zeros(self.nseq + 1, **i32)
            self.glob_pos = torch.zeros(max(T, 1), **i32)
        _lib.call("sc_index_build", self.cu_seqlens.data_ptr(), self.qgroup_len.data_ptr(), self.nseq,
                  T, self.tile_rows, self.qds_every if qds_positions is None else 0,
                  self.tok_seq.data_ptr(), self.tok_group.data_ptr(), self.tok_rel.data_ptr(),
                  self.tok_pos.data_ptr(), self.seq_tile_base.data_ptr(), self.seq_head_base.data_ptr(),
                  _lib.ptr(self.tok_flags) if qds_positions is None else None,
                  _lib.ptr(self.glob_cu) if qds_positions is None else None,
                  _lib.ptr(self.glob_pos) if qds_positions is None else None,
                  _lib.stream_handle(), exc=LayoutError)
        # host-side count of QDS global doc tokens (sizes the compact q/k/v copy)
        self.n_global = 0
        if self.qds_every:
            doc_tokens = self.group_lens_host[:, 2] - 1  # the doc group minus its final [SEP]
            self.n_global = int((doc_tokens // self.qds_every).sum())
        if qds_positions is not None:
            self._set_globals(qds_positions)
        self._ws = {}

    def _set_globals(self, positions_per_seq):
        """Explicit per-sequence global doc positions (AttentionPattern.global_positions)."""
        flags = np.zeros(self.total_tokens, np.uint8)
        cu = [0]
        pos = []
        for j, plist in enumerate(positions_per_seq):
            plist = sorted(set(int(p) for p in plist))
            start = self.cu_host[j] + 1 + self.qlen_host[j]
            for p in plist:
                if p >= self.group_lens_host[j, 2]:
                    raise LayoutError("global positions outside the document group")
                flags[start + p] = 1
            pos += plist
            cu.append(len(pos))
        self.qds_every = -1  # marks "globals present, explicit list"
        self.n_global = len(pos)
        self.tok_flags.copy_(torch.from_numpy(flags))
        self.glob_cu.copy_(torch.from_numpy(np.asarray(cu, np.int32)))
        if pos:
            self.glob_pos[: len(pos)].copy_(torch.from_numpy(np.asarray(pos, np.int32)))

    @classmethod
    def from_lengths(cls, seq_lens, qgroup_lens, device="cuda", tile_rows=DEFAULT_TILE_ROWS,
                     qds_every=0, qds_positions=None) -> "PackedLayout":
        seq_lens = np.asarray(seq_lens, dtype=np.int64)
        qgroup_lens = np.asarray(qgroup_lens, dtype=np.int64)
        if seq_lens.ndim != 1 or seq_lens.shape != qgroup_lens.shape or seq_lens.size == 0:
            raise LayoutError("seq_lens and qgroup_lens must be equal-length, non-empty 1-D")
        if np.any(qgroup_lens < 1) or np.any(seq_lens - 1 - qgroup_lens < 1):
            raise LayoutError("every sequence needs 1 cls row, >=1 query-group row and >=1 doc-group row")
        cu = np.zeros(seq_lens.size + 1, np.int64)
        np.cumsum(seq_lens, out=cu[1:])
        if cu[-1] >= 2**31:
            raise LayoutError("packed batch exceeds int32 token indexing")
        return cls(cu, qgroup_lens, device, tile_rows, qds_every, qds_positions)

    def attn_workspace(self, heads: int, head_dim: int, links: np.ndarray):
        key = (heads, head_dim, links.tobytes())
        if key not in self._ws:
            n = _lib.load().sc_attn_workspace_bytes_qds(self.nseq, self.total_tokens, heads, head_dim,
                                                        self.tile_rows, self.max_qgroup_len, links.ctypes.data,
                                                        self.n_global)
            # zeroed: the tail holds self-resetting per-sequence tile counters
            self._ws[key] = torch.zeros(n, dtype=torch.uint8, device=self.device) if n else None
        return self._ws[key]

    def mask(self, seq: int, pattern) -> np.ndarray:
        """Dense (s, s) bool mask of sequence ``seq`` exported by the device predicate (sc_mask_export)."""
        s = int(self.cu_host[seq + 1] - self.cu_host[seq])
        out = torch.empty(s * s, dtype=torch.uint8, device=self.device)
        links = pattern.links()
        _lib.call("sc_mask_export", self.cu_seqlens.data_ptr(), self.qgroup_len.data_ptr(), self.nseq,
                  seq, s, links.ctypes.data, _lib.ptr(self.tok_flags) if pattern.name == "qds" else None, out.data_ptr(),
                  _lib.stream_handle(), exc=LayoutError)
        return out.cpu().numpy().reshape(s, s).astype(bool)
