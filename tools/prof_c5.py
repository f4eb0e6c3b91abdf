"""cProfile the host side of a C5-shaped run (scaled): python tools/prof_c5.py N"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.run_configs as rc  # noqa: E402
import paper_1604_03570_b200 as tm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
tm.CONFIGS["C5"] = tm.CONFIGS["C5"].scaled(n, 32, 4)
cProfile.run("print(rc.heat_config('C5'))", "/tmp/c5.prof")
pstats.Stats("/tmp/c5.prof").sort_stats("cumulative").print_stats(30)
