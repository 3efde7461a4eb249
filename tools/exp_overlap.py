"""Does a hash draw on a side stream slow the one-wave C2 sketch kernel?
Times the sketch alone, the draw alone, and both overlapped, for several
phase-B grid caps.  Usage: python tools/exp_overlap.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native
from paper_1901_10559_b200._inputs import dense_operand

lib = _native.load()
I, R, L = 1_000_000, 2000, 100
a = torch.randn(I, R, dtype=torch.float64, device="cuda")
operand = dense_operand(a)
op = ids.CountSketchOp(I, L, seed=5, surjective=True)
op.bucket_index()
y = torch.empty((R, L), dtype=torch.float64, device="cuda")
side = torch.cuda.Stream()
main = torch.cuda.current_stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


def sketch():
    op.sketch_into(operand, y, flags=1)


def draw(seed):
    ids.CountSketchOp(I, L, seed=seed, surjective=True).bucket_index()


for _ in range(3):
    sketch()
    draw(1)
torch.cuda.synchronize()
for cap in (0, 64, 32, 16, 8):
    lib.ids_set_hash_grid_cap(cap)
    with torch.cuda.stream(side):
        draw(2)
    torch.cuda.synchronize()
    # alone
    a0, a1 = ev(), ev()
    a0.record(main); sketch(); a1.record(main)
    torch.cuda.synchronize()
    b0, b1 = ev(), ev()
    with torch.cuda.stream(side):
        b0.record(side); draw(3); b1.record(side)
    torch.cuda.synchronize()
    # overlapped: draw starts first on the side stream, then the sketch
    c0, c1, d0, d1 = ev(), ev(), ev(), ev()
    start = ev()
    start.record(main)
    side.wait_event(start)
    with torch.cuda.stream(side):
        d0.record(side); draw(4); d1.record(side)
    c0.record(main); sketch(); c1.record(main)
    torch.cuda.synchronize()
    # overlapped: sketch first, then the draw
    e0, e1, f0, f1 = ev(), ev(), ev(), ev()
    e0.record(main); sketch(); e1.record(main)
    side.wait_event(e0)
    with torch.cuda.stream(side):
        f0.record(side); draw(5); f1.record(side)
    torch.cuda.synchronize()
    print(f"cap {cap:3d}: sketch alone {a0.elapsed_time(a1)*1e3:7.0f} us, draw alone "
          f"{b0.elapsed_time(b1)*1e3:7.0f} us | draw-first: sketch {c0.elapsed_time(c1)*1e3:7.0f} "
          f"draw {d0.elapsed_time(d1)*1e3:7.0f} | sketch-first: sketch {e0.elapsed_time(e1)*1e3:7.0f} "
          f"draw {f0.elapsed_time(f1)*1e3:7.0f} (end {e0.elapsed_time(f1)*1e3:7.0f})", flush=True)
lib.ids_set_hash_grid_cap(0)
