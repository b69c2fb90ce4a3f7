"""Trajectories of the reference's toy trainer (pkg/src/qlrt/training.py:449-572)
for the GPU ToyModel / train_toy parity test: per-step losses and gradient
norms, initial / final eval loss.  Run in the build container, where the
reference imports:
    python tests/golden/make_golden_toy.py"""
import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from qlrt.training import TrainConfig, run_toy_training  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "toy_trajectories.json")
runs = []
for task, dtype, placement, lr, bs, steps, seed, dropout in (
        ("moons", "nf4", "all_linear", 0.01, 32, 60, 0, 0.0),
        ("moons", "fp4-e2m1", "qv_only", 0.01, 32, 60, 1, 0.0),
        ("moons", "nf4", "all_linear", 0.01, 32, 40, 2, 0.1),
        ("regression", "nf4", "all_linear", 3e-4, 128, 200, 0, 0.0),
        ("regression", "int4", "qv_only", 3e-4, 128, 100, 3, 0.0),
        ("regression", "fp32", "none", 3e-4, 128, 200, 1, 0.0)):
    cfg = TrainConfig(learning_rate=lr, batch_size=bs, steps=steps, seed=seed)
    r = run_toy_training(task, dtype, placement, cfg, dropout_p=dropout)
    runs.append({"task": task, "dtype": dtype, "placement": placement, "lr": lr, "batch_size": bs, "steps": steps,
                 "seed": seed, "dropout_p": dropout, "losses": list(r.losses), "grad_norms": list(r.grad_norms),
                 "initial_eval_loss": r.initial_eval_loss, "final_eval_loss": r.final_eval_loss})
with open(OUT, "w") as fh:
    json.dump(runs, fh)
print("wrote", OUT, len(runs), "runs")
