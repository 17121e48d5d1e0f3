"""(kernel selection / grid cap: TPCB_TRAIN_IMPL / TPCB_GRID_CAP env vars)
Reference acceptance criterion 6 on the GPU trainer: prints test MAPE / p90 for
training-kernel implementations and seeds.  python tools/crit6.py [impl ...]"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from conftest import load_golden  # noqa: E402
import paper_2311_09690_b200 as pb  # noqa: E402
from paper_2311_09690_b200 import _lib  # noqa: E402

g = load_golden("crit6")
off = np.concatenate([[0], np.cumsum(g["n_leaf"])])
samples, splits = [], {}
for i in range(len(g["n_leaf"])):
    comp = pb.CompactAst(g["vectors"][off[i]:off[i + 1]],
                         tuple(g["ordering"][off[i]:off[i + 1]].tolist()), (), int(g["n_leaf"][i]))
    s = pb.Sample(f"s{i}", f"t{g['task'][i]}", f"m{g['model'][i]}", "synth0", comp,
                  float(g["latency"][i]))
    samples.append(s)
    splits[s.id] = ("train", "valid", "test")[int(g["split"][i])]
ds = pb.Dataset(samples=samples, splits=splits)
devs = {"synth0": pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)}
test = ds.subset("test")
inputs = pb.encode_dataset(test, devs)
actual = np.array([s.latency_s for s in test])
impls = [int(a) for a in sys.argv[1:]] or [4]
for impl in impls:
    for seed in (0, 1, 2):
        res = pb.train(pb.desk_config(epochs=300, seed=seed), ds, devs)
        pred = pb.predict_batch(res.params, inputs, res.normalizer)
        rel = np.abs(pred - actual) / actual
        print(f"impl {impl} seed {seed}: test MAPE {pb.metrics(pred, actual)['mape']:.4f} "
              f"p90 {np.quantile(rel, 0.9):.4f} best val {res.best_val_mape:.4f} @ {res.best_epoch}",
              flush=True)
