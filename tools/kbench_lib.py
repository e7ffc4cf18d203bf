"""tools/kbench.py against another build of the library: python tools/kbench_lib.py <libname.so> [config]."""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_06635_b200 import binding as G

G.LIB_PATH = os.path.join(os.path.dirname(G.LIB_PATH), sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "kbench.py"), run_name="__main__")
