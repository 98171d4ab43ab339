"""Host cost of sincos_pairs_sharded: 8 shards of 2^16 angles on this device, launched from the
calling thread (the one-device path) or through the device's worker thread
(SINCOS_SHARDED_WORKERS=1, the multi-device path); µs per call, host side.
  python tools/shard_launch_cost.py; SINCOS_SHARDED_WORKERS=1 python tools/shard_launch_cost.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_cs_0406049_b200 as sp  # noqa: E402

G, n = 8, 1 << 16
shards = []
for g in range(G):
    t = torch.rand(n, device="cuda")
    shards.append({"theta": t, "sin": torch.empty_like(t), "cos": torch.empty_like(t)})
arr = sp._shard_array(shards)
L = sp.lib()
for _ in range(50):
    L.sincos_pairs_sharded(arr, G, 0)
torch.cuda.synchronize()
reps = 2000
t0 = time.perf_counter()
for _ in range(reps):
    L.sincos_pairs_sharded(arr, G, 0)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(json.dumps({"workers": os.environ.get("SINCOS_SHARDED_WORKERS", "0"), "shards": G,
                  "host_us_per_call": 1e6 * (t1 - t0) / reps, "host_us_per_shard": 1e6 * (t1 - t0) / reps / G}))
