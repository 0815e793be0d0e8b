"""Logit-ciphertext gather across ranks over NCCL (``heb_gather_logits``).

SURVEY.md §8e: image batches shard across GPUs with replicated keys and weights;
the one exchange is gathering the output logit ciphertexts.  The NCCL
communicator lives in libheb200 (C ABI); ``torch.distributed`` is only used to
hand the 128-byte NCCL unique id from rank 0 to the other ranks.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

ID_BYTES = 128


class LogitGather:
    """One NCCL communicator over ``world`` ranks on this rank's device."""

    def __init__(self, world: int, rank: int, device: int, share_id=None):
        """``share_id(bytes) -> bytes``: broadcast rank 0's id (default: torch.distributed)."""
        uid = ctypes.create_string_buffer(ID_BYTES)
        if rank == 0:
            _lib.call("heb_comm_unique_id", uid)
        raw = bytes(uid.raw)
        if world > 1:
            raw = (share_id or _broadcast_bytes)(raw)
        uid = ctypes.create_string_buffer(raw, ID_BYTES)
        handle = ctypes.c_void_p()
        _lib.call("heb_comm_init", ctypes.byref(handle), uid, world, rank, device)
        self.handle, self.world, self.rank = handle, world, rank
        self._comm_stream = None

    def gather(self, logits: torch.Tensor, stream=None) -> torch.Tensor:
        """(world, *logits.shape) on the device: every rank's logit ciphertexts.

        Ordered after ``stream``'s work (default: the current stream), and the caller's
        stream is ordered after the gather.  Collectives of one communicator must run in
        the same order on every rank, so all of them go through one communication stream
        even when several pipelines (streams) produce logits."""
        st = stream if stream is not None else torch.cuda.current_stream(logits.device)
        with torch.cuda.stream(st):  # the copy (if any) is ordered after the producer's work
            src = logits.contiguous()
        if self._comm_stream is None:
            self._comm_stream = torch.cuda.Stream(src.device)
        cs = self._comm_stream
        cs.wait_stream(st)
        with torch.cuda.stream(cs):
            out = torch.empty((self.world, *src.shape), dtype=src.dtype, device=src.device)
            _lib.call("heb_gather_logits", self.handle, src.data_ptr(), out.data_ptr(), src.numel(), cs.cuda_stream)
        src.record_stream(cs)
        out.record_stream(st)
        st.wait_stream(cs)
        return out

    def close(self) -> None:
        if self.handle:
            _lib.call("heb_comm_destroy", self.handle)
            self.handle = None


def _broadcast_bytes(raw: bytes) -> bytes:
    import torch.distributed as dist

    box = [raw]
    dist.broadcast_object_list(box, src=0)
    return box[0]
