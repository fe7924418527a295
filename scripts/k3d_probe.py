"""K3d (densify straight from the coded staging records) timed through the loader:
config-2-shaped procedural counts store (n_obs rows x 36k genes, HBM-resident coded
image), f=1024 B=16384 b=4096, densify f32 + normalize/log1p; prints the per-step
assembly kernel time (CUDA events around each launch) and its fraction of the
measured HBM peak by the bench's algorithmic bytes.  Product code only.

    python scripts/k3d_probe.py [--rows 500000] [--steps 40] [--out f32|bf16] [--no-norm]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2604_01949_b200 as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=500_000)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--out", default="f32")
    ap.add_argument("--no-norm", action="store_true")
    ap.add_argument("--staging", default="resident_coded")
    a = ap.parse_args()
    spec = (f"procedural:counts?n_obs={a.rows}&n_var=36000&seed=1&chunk_rows=1024&chunks_per_shard=128"
            f"&value_dtype=f32")
    reader = R.StoreReader(spec)
    man = reader.manifest()
    ds = R.DeviceStore(reader, 0, a.staging)
    rec_b, img_b = ds.image_bytes()
    st = torch.cuda.current_stream()
    it = R.BatchIterator(ds, R.LoaderConfig(1024, 16384, 4096, 0), 0, output="dense", out_dtype=a.out,
                         transform=None if a.no_norm else "normalize_log1p", out_slots=3, stream=st, time_kernels=True)
    for _ in range(5):
        it.next()
    torch.cuda.synchronize()
    c0 = it.counters()
    cells = 0
    for _ in range(a.steps):
        cells += it.next().n_rows
    torch.cuda.synchronize()
    c1 = it.counters()
    asm = (c1.assembly_ms - c0.assembly_ms) / a.steps
    esz = 2 if a.out == "bf16" else 4
    alg = cells / a.steps * (img_b / man.n_obs + 16 + man.n_var * esz + 8)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6500.0
    print(json.dumps({"assembly_us": asm * 1e3, "kernels_per_step": (c1.kernels_launched - c0.kernels_launched) / a.steps,
                      "GBps": alg / (asm / 1e3) / 1e9, "frac": alg / (asm / 1e3) / 1e9 / peak}))
    it.close()
    ds.close()


if __name__ == "__main__":
    main()
