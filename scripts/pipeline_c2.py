"""Whole reconstruction pipeline at a bench workload: index build, overlap search, host greedy merge."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1404_3456_b200 as rq
from bench import WORKLOADS
w = sys.argv[1] if len(sys.argv) > 1 else "c2"
G, L, k = WORKLOADS[w]
text, starts = rq.synth_read_text(G, L, k, 1, 2, pinned=True)
ex = rq.Executor(0)
fs = rq.fragment_set_from_text(text, starts)
rq.FragmentIndex(fs, ex).close()   # warm the arena
t0 = time.perf_counter(); ix = rq.FragmentIndex(fs, ex); ex.synchronize(); t1 = time.perf_counter()
ix.overlaps(20, reuse_buffers=True)
t1b = time.perf_counter(); ov = ix.overlaps(20, reuse_buffers=True); t2 = time.perf_counter()
sup, order = rq.greedy_superstring_from_overlaps(fs, ov); t3 = time.perf_counter()
print(f"{w}: k={k} n={text.size}  index {1e3*(t1-t0):.1f} ms  overlaps {1e3*(t2-t1b):.1f} ms ({ov.i.size} triples)  "
      f"host greedy merge {t3-t2:.2f} s -> superstring {len(sup)} bases from {order.size} reads (genome {G})")
genome = rq.synth_random_dna(G, 1).tobytes() if hasattr(rq, "synth_random_dna") else None
if genome is not None:
    print("superstring is a substring of the genome:", sup in genome, " covers", f"{len(sup)/G:.4f}", "of it")
