"""int8 tensor-core calibration: cuBLASLt (torch._int_mm) vs the repo's
tcgen05 int8 GEMM (qch_i8gemm_test, QCH_I8_BN) at large sizes, with the SM
clock sampled during the run.  python tools/i8_calib.py"""
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        out.append(r.stdout.strip())
        time.sleep(0.2)


def bench(fn, reps=20):
    import torch

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
    import torch

    from paper_2411_09982_b200 import _lib

    for (m, n, k) in [(8192, 8192, 8192), (4096, 4096, 32768)]:
        a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda")
        c = torch.empty(m, n, dtype=torch.int32, device="cuda")
        stop, smp = threading.Event(), []
        th = threading.Thread(target=clocks, args=(stop, smp))
        th.start()
        ms = bench(lambda: torch._int_mm(a, b.t()))
        ms2 = bench(lambda: _lib.call("qch_i8gemm_test", _lib.dptr(a), _lib.dptr(b), _lib.dptr(c), m, n, k,
                                      _lib.stream_ptr()))
        stop.set()
        th.join()
        f = 2.0 * m * n * k
        print(f"{m}x{n}x{k}: cuBLASLt int8 {f / ms / 1e9:.0f} TOPS ; repo tcgen05 i8 {f / ms2 / 1e9:.0f} TOPS ; "
              f"clocks/power {smp[len(smp) // 2] if smp else None} max {max(smp) if smp else None}", flush=True)
        x = torch.randn(m, k, dtype=torch.bfloat16, device="cuda")
        y = torch.randn(k, n, dtype=torch.bfloat16, device="cuda")
        ms3 = bench(lambda: x @ y)
        print(f"   bf16 cuBLAS {f / ms3 / 1e9:.0f} TFLOPS", flush=True)


if __name__ == "__main__":
    main()
