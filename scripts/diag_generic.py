"""Parity of the streamed vs the generic method at the metric shape (diagnostic)."""
import sys

sys.path.insert(0, ".")
from tests.test_gpu_layer import _oracle_subset_check  # noqa: E402

for method in ("stream", "generic"):
    for d in (1, 2, 3):
        try:
            f = _oracle_subset_check(1024, 64, 512, 4, d, channels=list(range(0, 512, 4)), seed=200 + d, method=method)
            print(method, d, "ok flips", f, flush=True)
        except AssertionError as e:
            print(method, d, "FAIL", str(e)[:300], flush=True)
