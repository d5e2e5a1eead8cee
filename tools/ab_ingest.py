"""Actor step + V/P ingest at c3 (bench.py's actor leg), for library A/B
(PQLG_LIB_VARIANT): prints the step time with and without the ingest."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = [sys.argv[0]]
import bench  # noqa: E402

args = bench.parse()
for rep in range(3):
    r = bench.run_actor(args, 0, 1, 0, 60, 5)
    print(f"rep {rep}: actor+ingest {r['ms_per_step'] * 1e3:.1f} us, "
          f"step only {r['actor_step_only']['ms_per_step'] * 1e3:.1f} us")
