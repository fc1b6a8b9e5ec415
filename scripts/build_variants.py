"""Build libwsgpu.so plus tuning variants: python scripts/build_variants.py name.so:DEF1,DEF2 ..."""
import os, sys; sys.path.insert(0, os.getcwd())
import sys
sys.path.insert(0, os.path.join(os.getcwd(), "paper_2409_03365_b200"))
import build  # noqa: E402  (not the package: its import loads the library)
build.build(force=True)
# spec: name.so:DEF1,DEF2[:nvcc flag;nvcc flag]
for spec in sys.argv[1:]:
    name, _, rest = spec.partition(':')
    defs, _, flags = rest.partition(':')
    build.build(force=True, defines=[d for d in defs.split(',') if d], name=name,
                extra_nvcc=[f for f in flags.split(';') if f])
