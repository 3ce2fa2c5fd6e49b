"""Run one bench variant alone (debugging aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

if __name__ == "__main__":
    name = sys.argv[1]
    if name == "ngram_kernel":
        from paper_2511_16193_b200 import _native
        print(bench.variant_ngram_kernel(_native.lib(), _native))
        for B, L in ((256, 1600), (256, 8192), (1024, 4096), (256, 32768)):
            print(B, L, bench.variant_ngram_kernel(_native.lib(), _native, B=B, L=L))
    if name == "configs4":
        print(bench.variant_configs4(graph="eager" not in sys.argv))
    if name == "configs2":
        print(bench.variant_configs2(graph="eager" not in sys.argv))
