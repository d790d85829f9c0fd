"""Probe the shared-memory layout + transaction bytes of a 16U4_ALIGN16B TMA load (W4A8 comparator)."""
import torch
from paper_2601_07475_b200 import arc

rows = 8
packed = torch.arange(rows * 64, dtype=torch.int32).remainder(256).to(torch.uint8)
# distinct nibbles: byte j of row r = (2*j) & 15 | ((2*j+1) & 15) << 4 pattern plus row tag
packed = torch.empty(rows, 64, dtype=torch.uint8)
for r in range(rows):
    for j in range(64):
        packed[r, j] = ((j % 16)) | (((r + j) % 16) << 4)
st, buf = arc.probe_u4_unpack(packed.cuda())
print("status", st.tolist())
for b in range(2):
    print("buf", b)
    for r in range(rows + 1):
        print(r, buf[b, r * 128:(r + 1) * 128].tolist())
print("src row0", packed[0].tolist())
print("src row1", packed[1].tolist())
