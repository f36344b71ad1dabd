"""Run bench.py against another build of libhmg.so (A/B on one box).
Usage: python tools/micro/bench_with_lib.py LIB.so [bench args...]"""
import os, runpy, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1605_00492_b200.binding as B
B._LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
