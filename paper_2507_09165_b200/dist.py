"""Multi-GPU plumbing (one process per GPU, torch.distributed for the process group).

* ``shard_range``: config c4 -- the global batch is sharded over ranks, no collective on the
  data path.
* ``rowpanel_tiles``: the upper 256-tiles a rank computes in the row-panel path (C ABI helper).
* ``RowPanelProjector``: config c5 -- one large n over P GPUs; every product of the chain is
  split by upper tiles over the ranks and the packed tiles are all-gathered over NCCL
  (psd_project_rowpanel).  The NCCL communicator is the library's own (libnccl.so.2, the copy
  torch loaded); its unique id travels through the torch.distributed process group.
"""
import ctypes

from ._lib import check, load


def shard_range(batch, world, rank):
    """[first, first + count) of the global batch owned by `rank` (contiguous, balanced)."""
    base, extra = divmod(batch, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def rowpanel_tiles(n, nranks, rank):
    """(codes, real_count): (I << 16) | J of the upper 256-tiles `rank` computes, in packed order."""
    lib = load()
    per = lib.psd_rowpanel_tiles(int(n), int(nranks), int(rank), None, 0)
    buf = (ctypes.c_uint32 * max(per, 1))()
    real = lib.psd_rowpanel_tiles(int(n), int(nranks), int(rank), buf, per)
    return [int(buf[i]) for i in range(per)], real


def broadcast_nccl_id(group=None):
    """Rank 0 creates an NCCL unique id; every rank returns the same 128 bytes."""
    import torch
    import torch.distributed as dist
    lib = load()
    raw = ctypes.create_string_buffer(128)
    if dist.get_rank(group) == 0:
        check(lib.psd_nccl_unique_id(raw), "psd_nccl_unique_id")
    t = torch.tensor(list(raw.raw), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


class RowPanelProjector:
    """P = psd_project over row panels of one n x n matrix on `world` GPUs (config c5)."""

    def __init__(self, flt, n, group=None):
        import torch.distributed as dist
        self.f = flt
        self.n = int(n)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.n % self.world:
            raise ValueError("n must be divisible by the number of ranks")
        self.rows = self.n // self.world
        uid = broadcast_nccl_id(group)
        self._lib = load()
        comm = ctypes.c_void_p()
        check(self._lib.psd_nccl_comm_create(uid, self.world, self.rank, ctypes.byref(comm)), "psd_nccl_comm_create")
        self.comm = comm

    def row_range(self):
        return self.rank * self.rows, self.rows

    def project(self, X_rows, out_rows=None, sign=False, stream=None):
        import torch
        from . import _stream_ptr
        if out_rows is None:
            out_rows = torch.empty_like(X_rows)
        assert X_rows.shape == (self.rows, self.n) and X_rows.is_contiguous() and X_rows.dtype == torch.float32
        check(self._lib.psd_project_rowpanel(self.f._h, ctypes.c_void_p(X_rows.data_ptr()), self.n, self.rank,
                                             self.world, ctypes.c_void_p(out_rows.data_ptr()), 1 if sign else 0,
                                             self.comm, _stream_ptr(stream)), "psd_project_rowpanel")
        return out_rows

    def close(self):
        if self.comm is not None and self.comm.value:
            self._lib.psd_nccl_comm_destroy(self.comm)
            self.comm = None
