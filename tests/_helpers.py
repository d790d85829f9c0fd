"""Test helpers shared by the GPU parity tests (no method arithmetic here)."""
import numpy as np
import torch

from _thirdparty import to_blocked


def valid_sf_mask(rows: int, Kp: int) -> np.ndarray:
    """Boolean mask over a roundup(rows,128)*Kp/16 scale buffer: True where the byte
    belongs to a valid row (< rows).  Derived from torch's to_blocked layout."""
    rp = (rows + 127) // 128 * 128
    src_row = torch.arange(rp, dtype=torch.int64)[:, None].expand(rp, Kp // 16).contiguous()
    return (to_blocked(src_row).reshape(-1) < rows).numpy()


def dev_bits(x: torch.Tensor):
    """bf16 tensor (any device) -> uint16 numpy bits on host."""
    return x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
