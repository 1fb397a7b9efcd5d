"""TEST INFRASTRUCTURE — ctypes binding of oracle/_ref/libprrtc_ref_io.so (the
reference's model_io.cpp + bench.cpp compiled in place, oracle/ref_io_capi.cpp).
Pins paper_2503_06757_b200/model_io.py and suite.py. Not product code."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2503_06757_b200._lib import Params

LIB = Path(__file__).resolve().parent / "_ref" / "libprrtc_ref_io.so"
DP = C.POINTER(C.c_double)
KIND = {"robot": 0, "scene": 1, "problem": 2, "path": 3}


def available() -> bool:
    return LIB.exists()


_CP = C.c_char_p
_I32P, _U32P, _U64P = C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
_REC = [C.c_uint32, C.POINTER(C.c_char_p), _I32P, _I32P, DP, DP, _U64P, _U64P, _U32P, _U64P]
_SIGS = {
    "refio_last_error": [_CP, C.c_size_t],
    "refio_roundtrip": [C.c_int, _CP, _CP],
    "refio_robot_dof": [_CP],
    "refio_problem_bundle": [_CP, C.POINTER(Params), C.POINTER(Params), _CP, C.c_size_t],
    "refio_problem_dir": [_CP, _CP, C.c_size_t],
    "refio_results_csv": _REC + [_CP, C.c_size_t],
    "refio_summarize_values": [DP, C.c_uint32, DP],
    "refio_summary_table": _REC + [_CP, C.c_size_t],
    "refio_ecdf": [C.c_uint32, _I32P, DP, DP, C.c_int, DP],
    "refio_apply_ablation": [_CP, _CP, C.POINTER(Params)],
    "refio_run_suite": [_CP, C.POINTER(Params), C.c_int, C.c_uint32, _U64P, _U32P, _U64P, _I32P, _I32P],
}


_CSV_CHILD = r"""
import ctypes as C, json, sys
lib = C.CDLL(sys.argv[1])
rows = json.loads(sys.stdin.read())
n = len(rows)
col = lambda t, i: (t * n)(*[r[i] for r in rows])
buf = C.create_string_buffer(1 << 22)
lib.refio_results_csv(C.c_uint32(n), (C.c_char_p * n)(*[r[0].encode() for r in rows]), col(C.c_int32, 1),
                      col(C.c_int32, 2), col(C.c_double, 3), col(C.c_double, 4), col(C.c_uint64, 5),
                      col(C.c_uint64, 6), col(C.c_uint32, 7), col(C.c_uint64, 8), buf, C.c_size_t(1 << 22))
sys.stdout.write(buf.value.decode())
"""


_SUITE_CHILD = r"""
import ctypes as C, json, sys
sys.path.insert(0, sys.argv[1].rsplit("/oracle/", 1)[0])
from paper_2503_06757_b200._lib import Params  # numpy-free
lib = C.CDLL(sys.argv[1])
base = Params()
for k, v in json.loads(sys.stdin.read()).items():
    setattr(base, k, int(v) if isinstance(v, bool) else v)
cap = 4096
h, w, s = (C.c_uint64 * cap)(), (C.c_uint32 * cap)(), (C.c_uint64 * cap)()
st, tr = (C.c_int32 * cap)(), (C.c_int32 * cap)()
n = lib.refio_run_suite(sys.argv[2].encode(), C.byref(base), int(sys.argv[3]), C.c_uint32(cap), h, w, s, st, tr)
if n < 0:
    b = C.create_string_buffer(4096)
    lib.refio_last_error(b, 4096)
    sys.exit(b.value.decode())
print(json.dumps([[h[i], w[i], s[i], st[i], tr[i]] for i in range(n)]))
"""


class RefIO:
    def __init__(self):
        self.lib = C.CDLL(str(LIB))
        for name, args in _SIGS.items():
            f = getattr(self.lib, name)
            f.argtypes = args
            f.restype = C.c_int

    def err(self) -> str:
        b = C.create_string_buffer(4096)
        self.lib.refio_last_error(b, 4096)
        return b.value.decode()

    def roundtrip(self, kind: str, src, dst):
        """reference load_* then write_*; returns None or the reference's error text."""
        rc = self.lib.refio_roundtrip(KIND[kind], str(src).encode(), str(dst).encode())
        return None if rc == 0 else self.err()

    def robot_dof(self, path) -> int:
        return self.lib.refio_robot_dof(str(path).encode())

    def problem_bundle(self, path, base):
        out = Params()
        name = C.create_string_buffer(1024)
        b = base.to_c()
        rc = self.lib.refio_problem_bundle(str(path).encode(), C.byref(b), C.byref(out), name, 1024)
        if rc != 0:
            raise RuntimeError(self.err())
        return out, name.value.decode()

    def problem_dir(self, d):
        buf = C.create_string_buffer(1 << 16)
        n = self.lib.refio_problem_dir(str(d).encode(), buf, 1 << 16)
        if n < 0:
            raise RuntimeError(self.err())
        return [x for x in buf.value.decode().split("\n") if x]

    @staticmethod
    def _rec_args(records):
        n = len(records)
        names = (C.c_char_p * n)(*[r.problem.encode() for r in records])
        arr = lambda t, v: (t * n)(*v)  # noqa: E731
        return [C.c_uint32(n), names, arr(C.c_int32, [r.trial for r in records]),
                arr(C.c_int32, [int(r.status) for r in records]), arr(C.c_double, [r.time_ms for r in records]),
                arr(C.c_double, [r.cost for r in records]), arr(C.c_uint64, [r.iterations for r in records]),
                arr(C.c_uint64, [r.sphere_tests for r in records]), arr(C.c_uint32, [r.workers for r in records]),
                arr(C.c_uint64, [r.seed for r in records])]

    def results_csv(self, records) -> str:
        """Run in a numpy-free child process: the reference's ostream integer
        insert crashes inside a process that has imported numpy (a libstdc++
        locale-facet clash in this image, not a reference bug)."""
        import json
        import subprocess
        import sys
        rows = [[r.problem, r.trial, int(r.status), r.time_ms, r.cost, r.iterations, r.sphere_tests, r.workers,
                 r.seed] for r in records]
        out = subprocess.run([sys.executable, "-c", _CSV_CHILD, str(LIB)], input=json.dumps(rows),
                             capture_output=True, text=True, check=True)
        return out.stdout

    def summary_table(self, records) -> str:
        buf = C.create_string_buffer(1 << 20)
        if self.lib.refio_summary_table(*self._rec_args(records), buf, 1 << 20) < 0:
            raise RuntimeError(self.err())
        return buf.value.decode()

    def summarize_values(self, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        out = np.zeros(7)
        if self.lib.refio_summarize_values(v.ctypes.data_as(DP), C.c_uint32(len(v)), out.ctypes.data_as(DP)) < 0:
            raise RuntimeError(self.err())
        return out

    def ecdf(self, statuses, time_ms, cost, use_cost: bool):
        n = len(statuses)
        st = np.ascontiguousarray(statuses, dtype=np.int32)
        t = np.ascontiguousarray(time_ms, dtype=np.float64)
        c = np.ascontiguousarray(cost, dtype=np.float64)
        out = np.zeros(2 * max(1, n))
        k = self.lib.refio_ecdf(C.c_uint32(n), st.ctypes.data_as(C.POINTER(C.c_int32)), t.ctypes.data_as(DP),
                                c.ctypes.data_as(DP), int(use_cost), out.ctypes.data_as(DP))
        return [(out[2 * i], out[2 * i + 1]) for i in range(k)]

    def apply_ablation(self, axis: str, value: str, params):
        p = params.to_c()
        if self.lib.refio_apply_ablation(axis.encode(), value.encode(), C.byref(p)) < 0:
            raise ValueError(self.err())
        return p

    def run_suite(self, d, base, trials: int):
        """reference run_suite over a problem directory (numpy-free child, see
        results_csv): (config_hash, workers, seed, status, trial) per record."""
        import json
        import subprocess
        import sys
        c = base.to_c()
        fields = {name: getattr(c, name) for name, _ in type(c)._fields_ if not name.startswith("_")}
        out = subprocess.run([sys.executable, "-c", _SUITE_CHILD, str(LIB), str(d), str(int(trials))],
                             input=json.dumps(fields), capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError(out.stderr.strip().splitlines()[-1] if out.stderr.strip() else "run_suite failed")
        return [tuple(r) for r in json.loads(out.stdout)]
