"""CPU tier: the host logic of multi-frequency batching --
the frequency-continuation driver (Algorithm 1) and the argument
checks of the concurrent batch entry points (no GPU compute)."""
import ctypes as C

import numpy as np
import pytest

from paper_1607_00968_b200 import _native, parallel
import paper_1607_00968_b200 as hz


def test_frequency_continuation_stages():
    seen = []

    def stage(m, omegas):
        seen.append(list(omegas))
        return m + 1.0

    models = parallel.frequency_continuation(np.zeros(3), [1.0, 2.0, 4.0], stage)
    assert seen == [[1.0], [1.0, 2.0], [1.0, 2.0, 4.0]]  # data of omega_1..omega_k at stage k
    assert [float(m[0]) for m in models] == [0.0, 1.0, 2.0, 3.0]  # warm start from the previous stage
    with pytest.raises(ValueError):
        parallel.frequency_continuation(np.zeros(3), [2.0, 1.0], stage)


def test_solve_blocks_multi_argument_checks():
    s = object()
    with pytest.raises(hz.ValidationError):
        hz.solve_blocks_multi([s, s], [np.zeros((4, 1)), np.zeros((4, 1))])
    with pytest.raises(hz.ValidationError):
        hz.solve_blocks_multi([s], [])
    assert hz.solve_blocks_multi([], []) == ([], [])
    L = _native.lib()
    assert L.hz_solve_blocks_multi(-1, None, None, None, None, None, None) == 1  # HZ_VALIDATION
    assert L.hz_solve_blocks_multi(0, None, None, None, None, None, None) == 0
    dup = (C.c_void_p * 2)(1234, 1234)
    n = (C.c_int64 * 2)(4, 4)
    k = (C.c_int * 2)(1, 1)
    p = (C.c_void_p * 2)(1, 1)
    assert L.hz_solve_blocks_multi(2, dup, n, k, p, p, None) == 1
    assert b"distinct" in L.hz_last_error_message()
