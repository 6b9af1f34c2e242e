"""Times pac_mask alone (hash + balancing) over N keys: keys/s and warp-instr budget."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen as dg
import paper_2603_15023_b200 as pac
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
w = dg.WORKLOADS["C2"]
keys = dg.device_column(w.pu, w.seed, 0, n)
out = torch.empty_like(keys)
for _ in range(3):
    pac.mask(keys, 12345, out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    pac.mask(keys, 12345, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"pac_mask: {n/ms/1e6:.3f} Gkeys/s, {ms:.3f} ms for {n} keys, {16*n/ms/1e6:.1f} GB/s")
