"""Throughput of the GPU .tns reader (qd_read_tns) against the reference's
read_tns (oracle/_ref, serial io.cpp) on the same synthetic file.

    python profiles/tns_bench.py [n_rows]   -> one JSON line
Both include canonicalisation (io.cpp:36-38).  The GPU figure is split into
the parse (device kernels, per-kernel time from the ncu launch list when run
under ncu) and the whole call (host text -> host rows, incl. H2D/D2H).
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2005_10427_b200 as qb  # noqa: E402


def make_text(n, dims, seed=1):
    rng = np.random.default_rng(seed)
    c = np.stack([rng.integers(1, d + 1, n) for d in dims], 1)
    v = rng.random(n)
    # fast formatting: numpy savetxt-like with repr-precision values
    lines = np.char.add(np.char.add(np.char.add(np.char.add(
        c[:, 0].astype(str), " "), c[:, 1].astype(str)), " "), c[:, 2].astype(str))
    vals = np.array([repr(x) for x in v.tolist()])
    return ("\n".join(np.char.add(np.char.add(lines, " "), vals).tolist()) + "\n").encode()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    text = make_text(n, [12092, 9184, 28818])
    ws = qb.Workspace(0)
    qb.read_tns_text(text[:100000].rsplit(b"\n", 2)[0] + b"\n", ws=ws)  # warm-up
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        t = qb.read_tns_text(text, ws=ws)
        ts.append(time.perf_counter() - t0)
    gpu_s = min(ts)
    out = {"what": "read_tns (canonicalised), GPU qd_read_tns vs reference io.cpp",
           "rows": n, "bytes": len(text), "gpu_call_s": round(gpu_s, 4),
           "gpu_mrows_s": round(n / gpu_s / 1e6, 1), "gpu_gb_s_text": round(len(text) / gpu_s / 1e9, 2)}
    from pyoracle import Reference, reference_available
    if reference_available():
        with tempfile.NamedTemporaryFile(suffix=".tns", delete=False) as f:
            f.write(text)
            path = f.name
        t0 = time.perf_counter()
        d, c, v = Reference().read_tns(path)
        ref_s = time.perf_counter() - t0
        os.unlink(path)
        out.update({"ref_s": round(ref_s, 3), "ref_mrows_s": round(n / ref_s / 1e6, 2),
                    "ref_cores": 1, "speedup_call": round(ref_s / gpu_s, 1),
                    "bit_exact_vs_ref": bool(np.array_equal(c, t.coords) and
                                             np.array_equal(v.view(np.uint64), t.values.view(np.uint64)))})
    # writer: write_tns of the tensor just read (text formatted on the GPU)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        wtext = qb.write_tns_text(t, ws=ws)
        ts.append(time.perf_counter() - t0)
    wpath = os.path.join(tempfile.gettempdir(), "qd_tns_bench_gpu.tns")
    tf = []
    for _ in range(3):
        t0 = time.perf_counter()
        qb.write_tns(t, wpath, ws=ws)
        tf.append(time.perf_counter() - t0)
    os.unlink(wpath)
    out.update({"write_gpu_text_s": round(min(ts), 4),
                "write_gpu_mrows_s": round(n / min(ts) / 1e6, 1),
                "write_gpu_file_s": round(min(tf), 4)})
    if reference_available():
        path = os.path.join(tempfile.gettempdir(), "qd_tns_bench_w.tns")
        t0 = time.perf_counter()
        Reference().write_tns(t.dims, t.coords, t.values, path)
        ref_w = time.perf_counter() - t0
        with open(path, "rb") as f:
            same = f.read() == bytes(wtext)
        os.unlink(path)
        out.update({"write_ref_s": round(ref_w, 3), "write_ref_mrows_s": round(n / ref_w / 1e6, 2),
                    "write_speedup_file": round(ref_w / min(tf), 1), "write_bytes_equal": same})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
