"""Timing of the LU step's full-matrix passes at n = 32768 (working copy,
max |A|): CUDA events on the launching stream, mean of 5 after a warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_23565_b200 import _dev, _lib  # noqa: E402
from paper_2509_23565_b200.matgen import generate_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = generate_device(0, n, seed=99, layout="F")
w = torch.empty_like(a)
bits = torch.zeros((2,), dtype=torch.int64, device="cuda")


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gb = 8.0 * n * n / 1e9
tc = t(lambda: _lib.call("oz_copy2d", a.data_ptr(), n, n, 1, n, w.data_ptr(), 1, n, _dev.stream()))
tm = t(lambda: _lib.call("oz_max_abs_bits", a.data_ptr(), n, n, 1, n, 0, bits.data_ptr(),
                         _dev.stream()))
print(f"n={n}: working copy {tc:.3f} ms ({2 * gb / tc:.0f} GB/s r+w), "
      f"max|A| {tm:.3f} ms ({gb / tm:.0f} GB/s)")
ref = float(torch.max(torch.abs(a)).item())
got = float(np.frombuffer(bits.cpu().numpy().tobytes()[:8], dtype=np.float64)[0])
print("max|A| exact:", got == ref, got, ref, "copy exact:", bool(torch.equal(a, w)))
