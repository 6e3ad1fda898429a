"""Debug helper: build the SA of a synthetic read set and report where it differs from the oracle."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import paper_1404_3456_b200 as rq
from oracle_lib import Oracle

G, L, k = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (50_000, 100, 5_000)
text, _ = rq.synth_read_text(G, L, k)
ex = rq.Executor(0)
got = rq.build_parallel(text, ex)
print("stats: init", got.stats.init_symbols, "rounds", got.stats.rounds, "passes", got.stats.sort_passes,
      "refined_global", got.stats.refined_global)
ora = Oracle()
wsa, _ = ora.build_sa(text)
bad = np.nonzero(got.sa != wsa)[0]
print("mismatches", bad.size, bad[:10])
