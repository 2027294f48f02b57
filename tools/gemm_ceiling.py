"""Engine ceiling: a large square DGEMM and tile-shaped segmented problems
through sdmrg_dgemm / the grouped engine (no sector irregularity)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2305_05581_b200 import _lib  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    lib = _lib.load()
    out = {}
    for n in (1024, 4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        c = torch.zeros(n, n, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def run():
            _lib.check(lib.sdmrg_dgemm(0, 0, n, n, n, 1.0, a.data_ptr(), n, b.data_ptr(), n, 0.0,
                                       c.data_ptr(), n, s))
        ms = timed(run)
        ref = (a.t() @ b.t()).t()
        err = (c - ref).abs().max().item() / ref.abs().max().item()
        out[f"dgemm_{n}"] = {"tflops": 2 * n ** 3 / ms / 1e9, "ms": ms, "relerr": err}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
