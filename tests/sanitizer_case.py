"""One small SMILE forward (and, for fp32, a training step) for compute-sanitizer runs
(tests/test_gpu_sanitizer.py): `python tests/sanitizer_case.py fp32|bf16 [peer]`."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import Case, assert_close_scaled  # noqa: E402


def main():
    dtype = sys.argv[1]
    peer = len(sys.argv) > 2 and sys.argv[2] == "peer"
    from paper_2212_05191_b200 import SmileLayer
    for mode in ("bilevel", "flat"):
        case = Case(2, 2, 2, 300, 64, 128, 1.0, dtype=dtype, mode=mode, dist="skewed", seed=91,
                    fused=(dtype == "bf16"))
        layer = SmileLayer(2, 2, 2, 64, 128, 300, 1.0, dtype, mode)
        if peer:
            layer.enable_peer_exchange()
        layer, out, loss, err = case.run_gpu(layer=layer)
        assert err == 0, err
        if dtype == "fp32":
            r = case.oracle_route()
            assert_close_scaled(out.float().cpu().numpy().reshape(-1, 64), case.oracle_out(r), 1e-5, mode)
        layer.close()
    print("SANITIZER_CASE_OK", flush=True)


if __name__ == "__main__":
    main()
