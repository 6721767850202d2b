"""Quick timing of a bounded fit (max_epochs) at a given size; prints ms/epoch."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import n2f_oracle as o
from paper_2108_10209_b200 import Engine, TrainConfig

size = int(sys.argv[1]) if len(sys.argv) > 1 else 512
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
impl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
clean = o.blob_rect_image(size, size, 0)
noisy = np.ascontiguousarray(o.gaussian_noisy(clean, 50 / 255, 1).astype(np.float32))
cfg = TrainConfig(seed=0, patience_epochs=10**6, avg_window=100, max_epochs=epochs)
eng = Engine(size, size, cfg, conv_impl=impl)
print("device bytes", eng.device_bytes / 2**30, "GiB")
for rep in range(2):
    t = time.perf_counter()
    out, r, hist, losses, secs = eng.fit_host(noisy)
    wall = time.perf_counter() - t
    print(f"size {size} epochs {r.epochs_run} gpu_ms {r.gpu_ms:.1f} -> {r.gpu_ms / r.epochs_run:.2f} ms/epoch; wall {wall:.2f}s; val {hist[:3]}")
