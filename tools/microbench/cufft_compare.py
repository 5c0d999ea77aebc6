"""Comparison baseline for the DFT stage (BJ north_star: "hand-written or cuFFT only as a comparison
baseline"): cuFFT (through torch.fft) on the full oversampled grids vs the library's pruned
box-only DFT stage, per MVM, for the BASELINE.json configurations.

The cuFFT side does what a textbook NFFT does between spreading and interpolation: a real-to-complex
FFT of every n_g^d grid (windows x RHS), the multiplier on the kept frequencies, and one complex-to-
real inverse per interpolated operator.  The multiply is omitted (it only favours cuFFT).

    python tools/microbench/cufft_compare.py            (on the GPU box)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402


def time_ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    dev = torch.device("cuda:0")
    out = {}
    for name in ("c1", "c2", "c3", "c4", "c5"):
        wl = workloads.CONFIGS[name]
        d = len(wl.windows[0])
        n_g = int(wl.N * wl.sigma_over)
        ops = len({"K" if o in ("K", "dsf") else o for o in wl.ops})
        batch = len(wl.windows) * wl.r
        shape = (batch,) + (n_g,) * d
        dims = tuple(range(1, d + 1))
        g = torch.randn(shape, dtype=torch.float64, device=dev)

        def step():
            spec = torch.fft.rfftn(g, dim=dims)
            for _ in range(ops):
                torch.fft.irfftn(spec, s=shape[1:], dim=dims)

        out[name] = {"grid": list(shape), "ops": ops, "cufft_ms_per_mvm": time_ms(step)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
