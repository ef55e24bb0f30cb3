"""Import-only stand-in for matplotlib (not installed in this image).

The reference package imports matplotlib at module import time
(subnewton/__init__.py -> bench.py -> plots.py); nothing on the hot path
renders figures.  This stub lets tests/golden/make_golden.py import the
unmodified reference to generate golden vectors.
"""


def use(*_args, **_kwargs):
    return None
