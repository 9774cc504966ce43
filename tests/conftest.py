import os
import sys

# BLAS-1 rounding in the Krylov setup depends on the OpenBLAS thread count; the
# golden fixtures were generated single-threaded (tests/golden/make_golden.py).
os.environ.setdefault('OPENBLAS_NUM_THREADS', '1')

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import pytest  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line('markers', 'gpu: needs a B200 (runs on the GPU box)')
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


@pytest.fixture(scope='session')
def golden():
    import numpy as np
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(ROOT, 'tests', 'golden', name + '.npz'),
                                       allow_pickle=False))
        return cache[name]
    return load
