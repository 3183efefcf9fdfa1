"""Build the bounds-checked library (FHT_CHECKS=1: every shared-memory access of the tile bodies, every
plain global store and TMA store coordinate checked; a violation prints and traps) as build/libfht_checks.so.
Run the GPU suite against it with FHT_LIB=build/libfht_checks.so (the stand-in for compute-sanitizer,
which is closed on this pool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
g.build(out=os.path.join(ROOT, "build", "libfht_checks.so"), extra_flags=["-DFHT_CHECKS=1"], load=False)
print("built build/libfht_checks.so")
