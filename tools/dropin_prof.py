"""(box) cProfile of the reference-compatible drop-in call on the headline batch."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2501_19042_b200 import SafetyFilter, SolverConfig, feasible_results  # noqa: E402

prob, shard, _ = bench.config2_case()
sf = SafetyFilter(prob, degree=10, config=SolverConfig(max_iters=500))
props = [x.copy() for x in shard]
sf.batch_solve(props[:8])
feasible_results(sf.batch_solve(props).results, prob)   # first full-size call: pinned staging buffers are cached
pr = cProfile.Profile()
pr.enable()
res = sf.batch_solve(props)
feasible_results(res.results, prob)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
