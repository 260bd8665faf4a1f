"""Trainer-export round trip golden, generated with the
REFERENCE trainer and engine (run in the build container, where
/root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_trainer_golden.py

Trains the reference trainer's 784-256-256-10 binary MLP
(pkg/trainer/src/bitnn_trainer/train.py:train_mlp) on the synthetic
MNIST-format set of tests/trainer_set.py, exports it with the trainer's own
writer (export.py:49-104) to trained_mlp.bdnn, and records the trainer's
float64 evaluation (train.py:135-156) and the reference engine's scores of
the test images (network.forward) in trainer.npz."""

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/trainer/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from bitnn.modelfile import load_model  # noqa: E402
from bitnn.network import Network, forward  # noqa: E402
from bitnn_trainer import evaluate, export, train_mlp  # noqa: E402
from trainer_set import make_set, write_idx  # noqa: E402

ARCH = (784, 256, 256, 10)

if __name__ == "__main__":
    tx, ty, vx, vy = make_set()
    with tempfile.TemporaryDirectory() as d:
        write_idx(d, tx, ty, vx, vy)
        state = train_mlp(ARCH, epochs=3, seed=0, data_dir=d)
    path = os.path.join(HERE, "trained_mlp.bdnn")
    export(state, path)
    preds, acc = evaluate(state, vx, vy)
    net = Network(load_model(path))
    scores = np.stack([forward(net, im.reshape(-1)).copy() for im in vx])
    np.savez_compressed(os.path.join(HERE, "trainer.npz"), trainer_preds=preds.astype(np.int64),
                        trainer_accuracy=np.float64(acc), engine_scores=scores)
    print(f"trainer accuracy {acc:.4f}; engine argmax agreement "
          f"{float(np.mean(np.argmax(scores, 1) == preds)):.4f}")
