"""Build libgscache.so into another file (A/B experiments on one GPU call):
  python tools/build_variant.py OUT.so [-DNAME=VALUE ...]   (extra nvcc flags)"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2507_19718_b200"))
import build  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
build.LIB = os.path.abspath(out)
if flags:
    src = build.sources
    build.sources = lambda: flags + src()
build.build(force=True)
print(build.LIB)
