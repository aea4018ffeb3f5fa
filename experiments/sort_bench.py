"""Device time of the hand-written radix sort (qvb_test_sort_bench)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2305_10863_b200 import qvb  # noqa: E402

for n in (1 << 20, 2_400_000, 16_000_000, 111_000_000):
    for bits in (22, 32, 50, 64):
        ms = C.c_double(0)
        qvb._check(qvb._lib().qvb_test_sort_bench(0, n, bits, 5, C.byref(ms)))
        print(f"n={n:>11d} bits={bits:2d}: {ms.value:8.3f} ms  {n / ms.value / 1e6:7.2f} G keys/s  "
              f"{n * 32 * ((bits + 7) // 8) / ms.value / 1e6:7.1f} GB/s (2R+2W of k,v per pass)")
