"""A/B timing of two builds of the native library on the same box (no claims).

    python tools/ab.py <lib.so> [prof.py args...]
"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_4297_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
script = os.environ.get("AB_SCRIPT", "prof.py")
sys.argv = [os.path.join(os.path.dirname(os.path.abspath(__file__)), script)] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
