"""Experiment timer (one GPU): HMult+Relin at batch B (argv[1], default 16)
and config-4 rotate, CUDA-event timed over 20 steps after 5 warm-up steps,
plus a bit check of every batch item against the oracle.  The library is
the one FHE_SM100_LIB names (tools/build_variant.sh variants).  Not a
benchmark: bench.py is."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    torch.cuda.set_device(0)
    w = bench.build_workload(B)
    step = lambda: bench.hmult_relin_step(w, B)  # noqa: E731
    ms = bench.time_steps(step, 20, 5, 1)
    bad = bench.check_batch_items(w, B)
    legs = bench.rotate_rescale_legs(w, B, 20, 5, 1)
    tag = os.path.basename(os.environ.get("FHE_SM100_LIB", "default"))
    print(f"{tag} {os.environ.get('FHE_FIN_STAGED', '')} hmult {B * 1000 / ms:.0f} ops/s "
          f"({ms:.3f} ms) bad={bad} rotate {legs['rotate']['ops_s']:.0f} "
          f"rescale {legs['rescale']['ops_s']:.0f}")


if __name__ == "__main__":
    main()
