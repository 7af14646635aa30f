"""Times trb_quantize_colors on real-valued samples (the device k-means path)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1310_3322_b200 import api
rng = np.random.default_rng(1)
for n, k, it in ((700, 16, 20), (20000, 16, 20), (200000, 32, 10)):
    px = np.ascontiguousarray(rng.uniform(0.0, 255.0, (n, 3)))
    api.quantize_colors(px, k, it, 3)
    t = time.perf_counter()
    for _ in range(3):
        api.quantize_colors(px, k, it, 3)
    print(f"n={n} k={k} iters={it}: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms")
