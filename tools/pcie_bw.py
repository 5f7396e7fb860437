"""PCIe copy bandwidth on this box: H2D / D2H alone, concurrently, and split
over two streams per direction (does a second copy engine add bandwidth?)."""
import torch

MB = 1 << 20
n = 48 * MB
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(h2d_streams, d2h_streams, reps=10):
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for st in streams:
        st.wait_event(ev0)
    for _ in range(reps):
        for i, st in enumerate(h2d_streams):
            part = n // len(h2d_streams)
            with torch.cuda.stream(st):
                d_in[i * part:(i + 1) * part].copy_(h_in[i * part:(i + 1) * part], non_blocking=True)
        for i, st in enumerate(d2h_streams):
            part = n // len(d2h_streams)
            with torch.cuda.stream(st):
                h_out[i * part:(i + 1) * part].copy_(d_out[i * part:(i + 1) * part], non_blocking=True)
    for st in streams:
        ev = torch.cuda.Event()
        ev.record(st)
        torch.cuda.current_stream().wait_event(ev)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    moved = n * ((1 if h2d_streams else 0) + (1 if d2h_streams else 0))
    return moved / ms / 1e6


s = streams
for name, a, b in [("H2D alone", [s[0]], []), ("D2H alone", [], [s[0]]),
                   ("H2D x2 streams", [s[0], s[1]], []), ("D2H x2 streams", [], [s[0], s[1]]),
                   ("H2D || D2H", [s[0]], [s[1]]),
                   ("H2D x2 || D2H x2", [s[0], s[1]], [s[2], s[3]])]:
    run(a, b)
    print(f"{name:>18}: {run(a, b):6.1f} GB/s total", flush=True)

# the pipeline's shapes: 3.4 MB query slabs in, 3 x 1.14 MB result rows out
# (one 2-D copy, pitch 8 n), interleaved on two streams
import ctypes as C  # noqa: E402
cud = C.CDLL("libcudart.so.12") if False else None
slab_in, row, pitch = 3_400_000, 1_140_000, 8_000_000
hq = torch.empty(24_000_000, dtype=torch.uint8, pin_memory=True)
dq = torch.empty(24_000_000, dtype=torch.uint8, device="cuda")
hres = torch.empty(3 * pitch, dtype=torch.uint8, pin_memory=True)
dres = torch.empty(3 * pitch, dtype=torch.uint8, device="cuda")


def pipeline(two_d, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s[0].wait_event(e0)
    s[1].wait_event(e0)
    for _ in range(reps):
        for k in range(7):
            with torch.cuda.stream(s[0]):
                dq[k * slab_in:(k + 1) * slab_in].copy_(hq[k * slab_in:(k + 1) * slab_in], non_blocking=True)
            with torch.cuda.stream(s[1]):
                if two_d:  # rows at pitch: a strided view copied as one 2-D copy
                    src = dres.view(3, pitch)[:, k * row:(k + 1) * row]
                    dst = hres.view(3, pitch)[:, k * row:(k + 1) * row]
                    dst.copy_(src, non_blocking=True)
                else:
                    for r in range(3):
                        hres[r * pitch + k * row:r * pitch + (k + 1) * row].copy_(
                            dres[r * pitch + k * row:r * pitch + (k + 1) * row], non_blocking=True)
    for st in (s[0], s[1]):
        ev = torch.cuda.Event()
        ev.record(st)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, (7 * slab_in + 21 * row) / ms / 1e6


for two_d in (False, True):
    pipeline(two_d)
    ms, bw = pipeline(two_d)
    print(f"pipeline shapes ({'2-D rows' if two_d else '1-D rows'}): {ms:.3f} ms per 24 + 24 MB, {bw:.1f} GB/s total",
          flush=True)
