"""Stub pyplot: any figure call fails loudly (rendering is out of scope)."""


def __getattr__(name):
    raise RuntimeError(f"matplotlib stub: pyplot.{name} is unavailable")
