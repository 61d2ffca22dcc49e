"""Development A/B builds: python tools/ab_build.py NAME [DEFINE ...] builds
build/ab/NAME.so with extra -D flags; run with PIRK_LIB=build/ab/NAME.so."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_10635_b200 import build as b

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "build", "ab", sys.argv[1] + ".so")
print(b.build(force=True, out=out, defines=sys.argv[2:]))
