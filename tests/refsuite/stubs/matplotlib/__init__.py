"""Presentation-only stand-in for matplotlib (absent from this image), used
solely by tests/refsuite so the reference's report module imports: figures
are written as empty PNG files. Nothing on the hot path touches it."""


def use(backend, *args, **kwargs):
    return None
