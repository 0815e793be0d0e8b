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

    def gather(self, logits: torch.Tensor, stream=None) -> torch.Tensor:
        """(world, *logits.shape) on the device: every rank's logit ciphertexts."""
        src = logits.contiguous()
        out = torch.empty((self.world, *src.shape), dtype=src.dtype, device=src.device)
        st = stream if stream is not None else torch.cuda.current_stream(src.device)
        _lib.call("heb_gather_logits", self.handle, src.data_ptr(), out.data_ptr(), src.numel(), st.cuda_stream)
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
