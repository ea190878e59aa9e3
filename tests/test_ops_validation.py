"""Host-side argument validation of the ops layer (no GPU needed): malformed
shapes / dtypes are rejected before anything reaches the C ABI, and CPU
tensors never run (there is no CPU fallback)."""
import pytest
import torch

from paper_2503_18292_b200 import ops


def test_paged_decode_rejects_bad_shapes():
    q = torch.zeros((4, 16, 128), dtype=torch.bfloat16)
    table = torch.zeros((4, 8), dtype=torch.int32)
    seq = torch.zeros(4, dtype=torch.int32)
    with pytest.raises(ValueError):  # out shape differs
        ops.paged_decode(None, None, 0, q, torch.zeros((4, 16, 64), dtype=torch.bfloat16), table, seq, 8, 16, 1.0)
    with pytest.raises(ValueError):  # fewer table rows than requests
        ops.paged_decode(None, None, 0, q, torch.empty_like(q), table[:2], seq, 8, 16, 1.0)
    with pytest.raises(TypeError):  # int64 block table
        ops.paged_decode(None, None, 0, q, torch.empty_like(q), table.long(), seq, 8, 16, 1.0)
    with pytest.raises(ValueError):  # not [B, Hq, D]
        ops.paged_decode(None, None, 0, q[0], torch.empty_like(q[0]), table, seq, 8, 16, 1.0)


def test_reshape_and_cache_rejects_bad_inputs():
    k = torch.zeros((6, 8, 128), dtype=torch.bfloat16)
    slots = torch.zeros(6, dtype=torch.int64)
    with pytest.raises(ValueError):  # too few slots
        ops.reshape_and_cache(None, None, k, k.clone(), slots[:3], 16)
    with pytest.raises(TypeError):  # key / value dtypes differ
        ops.reshape_and_cache(None, None, k, k.float(), slots, 16)
    with pytest.raises(TypeError):  # int32 slots
        ops.reshape_and_cache(None, None, k, k.clone(), slots.int(), 16)


def test_slot_mapping_and_cpu_tensors():
    table = torch.zeros((2, 4), dtype=torch.int32)
    req = torch.zeros(3, dtype=torch.int32)
    with pytest.raises(TypeError):  # int64 ordinals
        ops.slot_mapping(table, 4, req, req.long(), 16, torch.zeros(3, dtype=torch.int64))
    with pytest.raises(ValueError):  # out too small
        ops.slot_mapping(table, 4, req, req.clone(), 16, torch.zeros(2, dtype=torch.int64))
    with pytest.raises(ValueError, match="CUDA tensors only"):  # well-formed but on the CPU
        ops.slot_mapping(table, 4, req, req.clone(), 16, torch.zeros(3, dtype=torch.int64))


def test_prefill_rejects_bad_out():
    q = torch.zeros((10, 16, 256), dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        ops.paged_prefill(None, None, 0, q, torch.zeros((10, 8, 256), dtype=torch.bfloat16),
                          torch.tensor([0, 10], dtype=torch.int32), 10, torch.zeros((1, 4), dtype=torch.int32),
                          torch.zeros(1, dtype=torch.int32), 8, 16, 1.0)
