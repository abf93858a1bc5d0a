"""Host-side profile of Pipeline.process_stream (cProfile), 640x512 pinned frames."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1408_3526_b200 import Pipeline, default_params
from paper_1408_3526_b200.scenegen import SimConfig, generate_device

W, H = 640, 512
fr = generate_device(SimConfig(width=W, height=H, frame_count=1000), frames=32)
host = torch.empty((32, H, W), dtype=torch.float32, pin_memory=True)
host.copy_(fr)
hn = host.numpy()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
with Pipeline(default_params(), W, H) as pipe:
    for _ in pipe.process_stream(hn[i % 32] for i in range(40)):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in pipe.process_stream(hn[i % 32] for i in range(n)):
        pass
    dt = time.perf_counter() - t0
    print(f"plain: {dt / n * 1e3:.4f} ms/frame")
    pr = cProfile.Profile()
    pr.enable()
    for _ in pipe.process_stream(hn[i % 32] for i in range(n)):
        pass
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
