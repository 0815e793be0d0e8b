"""NCCL logit gather through the C ABI (heb_comm_* / heb_gather_logits).  The GPU box
has one device, so the communicator spans one rank: the all-gather must return the
rank's own logit words unchanged (the multi-rank exchange is the same NCCL call)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_single_rank_gather_is_identity():
    from paper_2102_00319_b200.comm import LogitGather

    g = LogitGather(1, 0, 0)
    try:
        x = torch.randint(0, 2**62, (10, 2, 3, 8192), dtype=torch.int64, device="cuda")
        out = g.gather(x)
        torch.cuda.synchronize()
        assert out.shape == (1, *x.shape)
        assert torch.equal(out[0], x)
    finally:
        g.close()


def test_gathered_logits_decrypt_like_local(tmp_path):
    """A gathered logit batch is bit-identical to the local one (raw residues travel)."""
    from paper_2102_00319_b200 import layers
    from paper_2102_00319_b200.backend import B200Backend, CipherBatch
    from paper_2102_00319_b200.comm import LogitGather
    from paper_2102_00319_b200.params import derive_params

    be = B200Backend(derive_params(1024, 300, 35, seed=7))
    keys = be.keygen()
    be.set_eval_key(keys)
    vals = np.random.default_rng(1).uniform(-1, 1, (4, be.slots))
    ct = be.encrypt_batch(vals, keys, np.arange(4))
    g = LogitGather(1, 0, 0)
    try:
        got = g.gather(ct.buf)[0]
    finally:
        g.close()
    dec = be.decrypt_batch(CipherBatch(got, ct.level, ct.scale, ct.noise_bits), keys)
    assert np.array_equal(dec, be.decrypt_batch(ct, keys))
    del layers


def test_gathers_from_several_pipeline_streams_keep_order():
    """Logits produced on different pipeline streams are gathered through one
    communication stream (NCCL collectives must run in issue order on every rank)."""
    from paper_2102_00319_b200.comm import LogitGather

    g = LogitGather(1, 0, 0)
    try:
        streams = [torch.cuda.Stream() for _ in range(3)]
        xs = [torch.full((4, 2, 3, 4096), i, dtype=torch.int64, device="cuda") for i in range(6)]
        outs = []
        for i, x in enumerate(xs):
            s = streams[i % 3]
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs.append(g.gather(x))
        torch.cuda.synchronize()
        assert all(torch.equal(o[0], x) for o, x in zip(outs, xs))
    finally:
        g.close()
