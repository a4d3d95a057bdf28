"""Device -> pinned-host copy bandwidth on this box (the e2e leg's ceiling).
Usage: python tools/pcie_bw.py  -> one line per copy pattern, GB/s."""
import torch

MB = 1 << 20
dev = torch.empty(64 * MB, dtype=torch.uint8, device="cuda")
host = torch.empty(64 * MB, dtype=torch.uint8, pin_memory=True)
frame = 5 * 640 * 480 * 20  # one config-1 frame of f32 rgb + depth + alpha


def bench(chunks, streams, reps=50):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    size = frame // chunks
    for _ in range(3):
        for k in range(chunks):
            with torch.cuda.stream(ss[k % streams]):
                host[k * size:(k + 1) * size].copy_(dev[k * size:(k + 1) * size], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:
        s.wait_event(e0)
    for _ in range(reps):
        for k in range(chunks):
            with torch.cuda.stream(ss[k % streams]):
                host[k * size:(k + 1) * size].copy_(dev[k * size:(k + 1) * size], non_blocking=True)
    for s in ss:
        e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return reps * chunks * size / (e0.elapsed_time(e1) / 1e3) / 1e9


for chunks, streams in [(1, 1), (15, 1), (15, 4), (60, 4)]:
    print(f"d2h {frame / 1e6:.1f} MB in {chunks} copies on {streams} stream(s): {bench(chunks, streams):.1f} GB/s")
