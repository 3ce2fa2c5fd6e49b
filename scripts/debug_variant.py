"""Run one bench variant alone (debugging aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

if __name__ == "__main__":
    name = sys.argv[1]
    if name == "configs2":
        print(bench.variant_configs2(graph="eager" not in sys.argv))
