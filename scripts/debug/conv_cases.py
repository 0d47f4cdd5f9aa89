"""Run conv variants one per process at a small size; report which fail.
usage: python scripts/debug/conv_cases.py [width height] -> one line per config"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

def one(i, w, h):
    import numpy as np
    import benchmarks_oracle as bo
    from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
    b = benchmark("conv", width=w, height=h)
    src = CudaMeasurementSource(b)
    hst = b.host_inputs()
    want, mag = bo.conv(hst["in"], hst["filt"])
    err = bo.within(src.output(i), want, mag, 1.0)
    print("cfg", i, b.values(i), "smem", b.smem_bytes(b.values(i)), "err", err, flush=True)

if __name__ == "__main__":
    if sys.argv[1] == "one":
        one(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])); sys.exit(0)
    w, h = int(sys.argv[1]), int(sys.argv[2])
    from paper_2102_05297_b200.live import benchmark
    b = benchmark("conv", width=w, height=h)
    n = len(b.space)
    idxs = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else range(0, n, max(1, n // 60))
    for i in idxs:
        r = subprocess.run([sys.executable, __file__, "one", str(i), str(w), str(h)],
                           capture_output=True, text=True, timeout=300)
        line = (r.stdout.strip().splitlines() or [""])[-1]
        print(i, "rc", r.returncode, line if r.returncode == 0 else r.stderr.strip().splitlines()[-1][:300], flush=True)
