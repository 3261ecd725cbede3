"""A/B: run tools/latency.py-style timing for an alternate build of the library (path in argv[1])."""
import os, sys, shutil
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_04471_b200 as sr
from paper_1609_04471_b200 import build as b
b.LIB = sys.argv[1]
b.needs_build = lambda: False
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "latency.py")).read())
