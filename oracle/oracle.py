"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracles.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module, and only as the checker / baseline.  Nothing in
``paper_2601_09951_b200`` imports it.

Two libraries:

* ``ORC``  — ``oracle/libvqf_oracle.so``: the plain-C restatement
  (``vqf_oracle.c``), each function citing the reference file:line it follows.
* ``REF``  — ``oracle/_ref/libvqf_ref.so``: the UNMODIFIED reference headers
  (``/root/reference/proj/include/vqeforge``) compiled against
  ``oracle/eigen_shim`` behind ``ref_capi.cpp``.  Present when it was built in
  the container (it then travels to the GPU box as a prebuilt file).

Both speak the same sparse-CSR Hamiltonian form as the product's C ABI
(``include/vqf_b200.h``): coeffs (re, im) per term, offsets, qubits, axes
(1 X, 2 Y, 3 Z).
"""
from __future__ import annotations

import ctypes as C
import os
import random
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "libvqf_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libvqf_ref.so")

ERR_TYPES = {1: ValueError, 2: RuntimeError, 3: AssertionError, 4: ArithmeticError, 9: Exception}
AXIS = {"X": 1, "Y": 2, "Z": 3}
AXIS_CHR = "IXYZ"

_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)


@dataclass
class Ham:
    """A QubitHamiltonian (pauli.hpp:116-129): terms = [(complex, [(q, axis)])]."""

    n_qubits: int
    terms: list = field(default_factory=list)

    def csr(self):
        coeffs = np.zeros(2 * max(1, len(self.terms)), dtype=np.float64)
        offsets = np.zeros(len(self.terms) + 1, dtype=np.uint32)
        qs, axs = [], []
        for t, (c, axes) in enumerate(self.terms):
            coeffs[2 * t] = complex(c).real
            coeffs[2 * t + 1] = complex(c).imag
            for q, a in axes:
                qs.append(q)
                axs.append(a if isinstance(a, int) else AXIS[a])
            offsets[t + 1] = len(qs)
        qubits = np.array(qs if qs else [0], dtype=np.uint32)
        axes_ = np.array(axs if axs else [0], dtype=np.uint8)
        return coeffs, offsets, qubits, axes_

    def key(self, t):
        return "".join(f"{AXIS_CHR[a]}{q}" for q, a in self.terms[t][1])

    def to_text(self) -> str:
        """pauli.hpp:294-309 (%.17g; Python repr round-trips identically)."""
        lines = []
        for c, axes in self.terms:
            s = f"{_g17(c.real)} {_g17(c.imag)}"
            if axes:
                s += " " + "".join(f"{AXIS_CHR[a]}{q}" for q, a in axes)
            lines.append(s)
        return "".join(line + "\n" for line in lines)

    @staticmethod
    def from_text(n_qubits: int, text: str) -> "Ham":
        terms = []
        for line in text.splitlines():
            parts = line.split()
            if not parts:
                continue
            re_, im_ = float(parts[0]), float(parts[1])
            axes = []
            if len(parts) > 2:
                s = parts[2]
                i = 0
                while i < len(s):
                    a = AXIS[s[i]]
                    j = i + 1
                    while j < len(s) and s[j].isdigit():
                        j += 1
                    axes.append((int(s[i + 1 : j]), a))
                    i = j
            terms.append((complex(re_, im_), axes))
        return Ham(n_qubits, terms)


def _g17(x: float) -> str:
    return "%.17g" % x


class _HamOut:
    def __init__(self, cap_terms=8192, cap_axes=1 << 18):
        self.nt = C.c_uint32()
        self.coeffs = np.zeros(2 * cap_terms, dtype=np.float64)
        self.offsets = np.zeros(cap_terms + 1, dtype=np.uint32)
        self.qubits = np.zeros(cap_axes, dtype=np.uint32)
        self.axes = np.zeros(cap_axes, dtype=np.uint8)
        self.cap_terms, self.cap_axes = cap_terms, cap_axes

    def args(self):
        return (
            C.byref(self.nt),
            self.coeffs.ctypes.data_as(_dp),
            self.offsets.ctypes.data_as(_u32p),
            self.qubits.ctypes.data_as(_u32p),
            self.axes.ctypes.data_as(_u8p),
            C.c_uint32(self.cap_terms),
            C.c_uint32(self.cap_axes),
        )

    def ham(self, n_qubits) -> Ham:
        terms = []
        for t in range(self.nt.value):
            lo, hi = int(self.offsets[t]), int(self.offsets[t + 1])
            axes = [(int(self.qubits[k]), int(self.axes[k])) for k in range(lo, hi)]
            terms.append((complex(self.coeffs[2 * t], self.coeffs[2 * t + 1]), axes))
        return Ham(n_qubits, terms)


def _check(rc, err):
    if rc:
        raise ERR_TYPES.get(rc, Exception)(err.value.decode())


def _ham_in(h: Ham):
    coeffs, offsets, qubits, axes = h.csr()
    keep = (coeffs, offsets, qubits, axes)
    return keep, (
        C.c_uint32(h.n_qubits),
        C.c_uint32(len(h.terms)),
        coeffs.ctypes.data_as(_dp),
        offsets.ctypes.data_as(_u32p),
        qubits.ctypes.data_as(_u32p),
        axes.ctypes.data_as(_u8p),
    )


# --------------------------------------------------------------------- REF
class Reference:
    """The reference's own CPU path (oracle/_ref/libvqf_ref.so)."""

    def __init__(self, path=REF_PATH):
        self.lib = C.CDLL(path)
        self.err = C.create_string_buffer(4096)

    def _e(self):
        return self.err, C.c_size_t(len(self.err))

    def build_h2_hamiltonian(self, d: float) -> Ham:
        o = _HamOut()
        _check(self.lib.ref_build_h2_hamiltonian(C.c_double(d), *o.args(), *self._e()), self.err)
        return o.ham(4)

    def hartree_fock(self, d: float):
        out = (C.c_double * 4)()
        _check(self.lib.ref_hartree_fock(C.c_double(d), out, *self._e()), self.err)
        return {"hf_energy": out[0], "electronic": out[1], "nuclear": out[2], "scf_iterations": int(out[3])}

    def build_tfim(self, n, coupling=1.0, fld=1.0) -> Ham:
        o = _HamOut()
        _check(self.lib.ref_build_tfim(C.c_uint32(n), C.c_double(coupling), C.c_double(fld), *o.args(), *self._e()), self.err)
        return o.ham(n)

    def build_z_sum(self, n) -> Ham:
        o = _HamOut()
        _check(self.lib.ref_build_z_sum(C.c_uint32(n), *o.args(), *self._e()), self.err)
        return o.ham(n)

    def canonicalize(self, h: Ham) -> Ham:
        o = _HamOut()
        keep, args = _ham_in(h)
        _check(self.lib.ref_canonicalize(*args, *o.args(), *self._e()), self.err)
        return o.ham(h.n_qubits)

    def to_text(self, h: Ham) -> str:
        buf = C.create_string_buffer(1 << 20)
        keep, args = _ham_in(h)
        _check(self.lib.ref_to_text(*args, buf, C.c_size_t(len(buf)), *self._e()), self.err)
        return buf.value.decode()

    def exact_ground_energy(self, h: Ham) -> float:
        out = C.c_double()
        keep, args = _ham_in(h)
        _check(self.lib.ref_exact_ground_energy(*args, C.byref(out), *self._e()), self.err)
        return out.value

    def apply_gates(self, n, amps: np.ndarray, gates) -> np.ndarray:
        """gates: list of (kind, angle, wires). Returns new complex128 array."""
        a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
        G = len(gates)
        kinds = np.array([g[0] for g in gates] or [0], dtype=np.int32)
        angles = np.array([g[1] for g in gates] or [0.0], dtype=np.float64)
        nw = np.array([len(g[2]) for g in gates] or [0], dtype=np.uint32)
        w4 = np.zeros(4 * max(G, 1), dtype=np.uint32)
        for i, g in enumerate(gates):
            w4[4 * i : 4 * i + len(g[2])] = g[2]
        _check(
            self.lib.ref_apply_gates(
                C.c_uint32(n), a.ctypes.data_as(_dp), C.c_uint32(G), kinds.ctypes.data_as(C.POINTER(C.c_int)),
                angles.ctypes.data_as(_dp), nw.ctypes.data_as(_u32p), w4.ctypes.data_as(_u32p), *self._e()
            ),
            self.err,
        )
        return a

    def expectation(self, n, amps, h: Ham) -> float:
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        out = C.c_double()
        keep, args = _ham_in(h)
        _check(self.lib.ref_expectation(C.c_uint32(n), a.ctypes.data_as(_dp), *args, C.byref(out), *self._e()), self.err)
        return out.value

    # ---- the reference's own seeded fixtures (tests/test_helpers.hpp:28-69)
    def random_hamiltonian(self, seed: int, n: int, n_terms: int, real=True) -> Ham:
        """testutil::random_hamiltonian(std::mt19937(seed), n, T, real): the
        exact Pauli sum the reference's tests draw (uncanonicalised)."""
        o = _HamOut(cap_terms=max(8192, n_terms), cap_axes=max(1 << 18, n_terms * n))
        _check(self.lib.ref_random_hamiltonian(C.c_uint32(seed), C.c_uint32(n), C.c_int(n_terms), C.c_int(int(real)),
                                               *o.args(), *self._e()), self.err)
        return o.ham(n)

    def random_state(self, seed: int, n: int) -> np.ndarray:
        """testutil::random_state(std::mt19937(seed), n), bit for bit."""
        a = np.empty(1 << n, dtype=np.complex128)
        _check(self.lib.ref_random_state(C.c_uint32(seed), C.c_uint32(n), a.ctypes.data_as(_dp), *self._e()), self.err)
        return a

    # ---- CPU baselines (bench.py): one reference call on a resident state
    def time_apply_gate(self, n, amps, kind, angle, wires, reps=1) -> float:
        """Best-of-reps seconds of ONE statevector.hpp:148 apply_gate call
        (single-threaded, as the reference is); amps are updated in the
        reference's own copy only."""
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        w = (C.c_uint32 * 4)(*(list(wires) + [0] * (4 - len(wires))))
        out = C.c_double()
        _check(self.lib.ref_time_apply_gate(C.c_uint32(n), a.ctypes.data_as(_dp), C.c_int(kind), C.c_double(angle),
                                            C.c_uint32(len(wires)), w, C.c_int(reps), C.byref(out), *self._e()), self.err)
        return out.value

    def time_expectation(self, n, amps, h: Ham, reps=1):
        """(value, best-of-reps seconds) of ONE statevector.hpp:217 call."""
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        val, sec = C.c_double(), C.c_double()
        keep, args = _ham_in(h)
        _check(self.lib.ref_time_expectation(C.c_uint32(n), a.ctypes.data_as(_dp), *args, C.c_int(reps), C.byref(val),
                                             C.byref(sec), *self._e()), self.err)
        return val.value, sec.value

    def prepare_ansatz(self, kind, layers, theta, n):
        t = np.ascontiguousarray(theta, dtype=np.float64)
        a = np.zeros(1 << n, dtype=np.complex128)
        _check(
            self.lib.ref_prepare_ansatz(C.c_int(kind), C.c_uint32(layers), t.ctypes.data_as(_dp), C.c_uint32(len(t)),
                                        C.c_uint32(n), a.ctypes.data_as(_dp), *self._e()),
            self.err,
        )
        return a

    def energy(self, kind, layers, theta, h: Ham) -> float:
        t = np.ascontiguousarray(theta, dtype=np.float64)
        out = C.c_double()
        keep, args = _ham_in(h)
        _check(self.lib.ref_energy(C.c_int(kind), C.c_uint32(layers), t.ctypes.data_as(_dp), C.c_uint32(len(t)), *args,
                                   C.byref(out), *self._e()), self.err)
        return out.value

    def gradient(self, kind, layers, theta, h: Ham):
        t = np.ascontiguousarray(theta, dtype=np.float64)
        out = np.zeros(len(t), dtype=np.float64)
        keep, args = _ham_in(h)
        _check(self.lib.ref_gradient(C.c_int(kind), C.c_uint32(layers), t.ctypes.data_as(_dp), C.c_uint32(len(t)), *args,
                                     out.ctypes.data_as(_dp), *self._e()), self.err)
        return out

    def run_vqe(self, h: Ham, kind=0, layers=0, lr=0.01, b1=0.9, b2=0.999, eps=1e-8, max_iter=200, tol=None, init=()):
        P = 1 if kind == 0 else layers * h.n_qubits
        init = np.ascontiguousarray(init, dtype=np.float64)
        theta = np.zeros(P, dtype=np.float64)
        traj = np.zeros(max_iter + 1, dtype=np.float64)
        e, tl, it, ev, wall = C.c_double(), C.c_uint32(), C.c_int(), C.c_uint64(), C.c_double()
        keep, args = _ham_in(h)
        _check(
            self.lib.ref_run_vqe(
                *args, C.c_int(kind), C.c_uint32(layers), C.c_double(lr), C.c_double(b1), C.c_double(b2), C.c_double(eps),
                C.c_int(max_iter), C.c_int(tol is not None), C.c_double(tol or 0.0), init.ctypes.data_as(_dp),
                C.c_uint32(len(init)), C.byref(e), theta.ctypes.data_as(_dp), traj.ctypes.data_as(_dp), C.byref(tl),
                C.byref(it), C.byref(ev), C.byref(wall), *self._e()
            ),
            self.err,
        )
        return {"energy": e.value, "theta": theta, "trajectory": traj[: tl.value].copy(), "iterations_run": it.value,
                "circuit_evaluations": ev.value, "wall_seconds": wall.value}

    def bond_grid(self, d_min, d_max, n):
        out = np.zeros(max(n, 1), dtype=np.float64)
        _check(self.lib.ref_bond_grid(C.c_double(d_min), C.c_double(d_max), C.c_int(n), out.ctypes.data_as(_dp), *self._e()), self.err)
        return out

    def split_chunks(self, n_items, n_chunks):
        out = np.zeros(2 * max(n_chunks, 1), dtype=np.uint64)
        _check(self.lib.ref_split_chunks(C.c_uint64(n_items), C.c_uint64(n_chunks), out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                         *self._e()), self.err)
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n_chunks)]

    def effective_workers(self, requested):
        out = C.c_int()
        _check(self.lib.ref_effective_workers(C.c_int(requested), C.byref(out), *self._e()), self.err)
        return out.value

    def run_sweep(self, d_min=0.1, d_max=3.0, n_points=100, workers=1, lr=0.01, b1=0.9, b2=0.999, eps=1e-8,
                  max_iter=200, tol=None):
        n = n_points
        bond, energy, theta, wall = (np.zeros(max(n, 1)) for _ in range(4))
        iters, ok = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
        stride = 256
        errors = C.create_string_buffer(stride * max(n, 1))
        per_worker = np.zeros(max(workers, 1))
        total, all_ok = C.c_double(), C.c_int()
        ip = C.POINTER(C.c_int)
        _check(
            self.lib.ref_run_sweep(
                C.c_double(d_min), C.c_double(d_max), C.c_int(n), C.c_int(workers), C.c_double(lr), C.c_double(b1),
                C.c_double(b2), C.c_double(eps), C.c_int(max_iter), C.c_int(tol is not None), C.c_double(tol or 0.0),
                bond.ctypes.data_as(_dp), energy.ctypes.data_as(_dp), theta.ctypes.data_as(_dp), iters.ctypes.data_as(ip),
                wall.ctypes.data_as(_dp), ok.ctypes.data_as(ip), errors, C.c_size_t(stride), per_worker.ctypes.data_as(_dp),
                C.byref(total), C.byref(all_ok), *self._e()
            ),
            self.err,
        )
        errs = [errors.raw[i * stride : (i + 1) * stride].split(b"\0", 1)[0].decode() for i in range(n)]
        return {"bond": bond[:n], "energy": energy[:n], "theta": theta[:n], "iterations": iters[:n], "wall": wall[:n],
                "ok": ok[:n].astype(bool), "errors": errs, "per_worker_seconds": per_worker, "total_wall_seconds": total.value,
                "all_ok": bool(all_ok.value)}

    def run_scaling_study(self, widths, layers=2, iterations=5, lr=0.05, coupling=1.0, fld=1.0, z_sum=False,
                          theta_init=0.1, force=False):
        w = np.ascontiguousarray(widths, dtype=np.uint32)
        k = len(w)
        sb = np.zeros(k, dtype=np.uint64)
        rt, fe = np.zeros(k), np.zeros(k)
        it = np.zeros(k, dtype=np.int32)
        _check(
            self.lib.ref_run_scaling_study(
                w.ctypes.data_as(_u32p), C.c_uint32(k), C.c_uint32(layers), C.c_int(iterations), C.c_double(lr),
                C.c_double(coupling), C.c_double(fld), C.c_int(int(z_sum)), C.c_double(theta_init), C.c_int(int(force)),
                sb.ctypes.data_as(C.POINTER(C.c_uint64)), rt.ctypes.data_as(_dp), fe.ctypes.data_as(_dp),
                it.ctypes.data_as(C.POINTER(C.c_int)), *self._e()
            ),
            self.err,
        )
        return [{"n_qubits": int(w[i]), "state_bytes": int(sb[i]), "runtime_seconds": float(rt[i]),
                 "final_energy": float(fe[i]), "iterations_run": int(it[i])} for i in range(k)]


# --------------------------------------------------------------------- ORC
class _OrcHam(C.Structure):
    _fields_ = [("n_qubits", C.c_uint32), ("n_terms", C.c_uint32), ("coeffs", _dp), ("offsets", _u32p),
                ("qubits", _u32p), ("axes", _u8p)]


class _OrcHamOut(C.Structure):
    _fields_ = [("n_terms", _u32p), ("coeffs", _dp), ("offsets", _u32p), ("qubits", _u32p), ("axes", _u8p),
                ("cap_terms", C.c_uint32), ("cap_axes", C.c_uint32)]


class _OrcGate(C.Structure):
    _fields_ = [("kind", C.c_int), ("angle", C.c_double), ("n_wires", C.c_uint32), ("wires", C.c_uint32 * 4)]


class _OrcAdam(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double),
                ("max_iterations", C.c_int), ("has_tolerance", C.c_int), ("gradient_tolerance", C.c_double)]


class _OrcVqeResult(C.Structure):
    _fields_ = [("energy", C.c_double), ("theta", _dp), ("trajectory", _dp), ("traj_len", C.c_uint32),
                ("iterations_run", C.c_int), ("circuit_evaluations", C.c_uint64)]


class Oracle:
    """The C restatement (oracle/libvqf_oracle.so)."""

    def __init__(self, path=ORC_PATH):
        self.lib = C.CDLL(path)
        self.lib.orc_n_parameters.restype = C.c_uint32
        self.err = C.create_string_buffer(4096)

    def _e(self):
        return self.err, C.c_size_t(len(self.err))

    @staticmethod
    def _ham(h: Ham):
        coeffs, offsets, qubits, axes = h.csr()
        s = _OrcHam(h.n_qubits, len(h.terms), coeffs.ctypes.data_as(_dp), offsets.ctypes.data_as(_u32p),
                    qubits.ctypes.data_as(_u32p), axes.ctypes.data_as(_u8p))
        return (coeffs, offsets, qubits, axes), s

    @staticmethod
    def _out():
        o = _HamOut()
        s = _OrcHamOut(C.pointer(o.nt), o.coeffs.ctypes.data_as(_dp), o.offsets.ctypes.data_as(_u32p),
                       o.qubits.ctypes.data_as(_u32p), o.axes.ctypes.data_as(_u8p), o.cap_terms, o.cap_axes)
        return o, s

    def canonicalize(self, h: Ham) -> Ham:
        keep, hs = self._ham(h)
        o, os_ = self._out()
        _check(self.lib.orc_canonicalize(C.byref(hs), C.byref(os_), *self._e()), self.err)
        return o.ham(h.n_qubits)

    def build_h2_hamiltonian(self, d) -> Ham:
        o, os_ = self._out()
        _check(self.lib.orc_build_h2_hamiltonian(C.c_double(d), C.byref(os_), *self._e()), self.err)
        return o.ham(4)

    def hartree_fock(self, d):
        out = (C.c_double * 4)()
        _check(self.lib.orc_hartree_fock(C.c_double(d), out, *self._e()), self.err)
        return {"hf_energy": out[0], "electronic": out[1], "nuclear": out[2], "scf_iterations": int(out[3])}

    def build_tfim(self, n, coupling=1.0, fld=1.0) -> Ham:
        o, os_ = self._out()
        _check(self.lib.orc_build_tfim(C.c_uint32(n), C.c_double(coupling), C.c_double(fld), C.byref(os_), *self._e()), self.err)
        return o.ham(n)

    def build_z_sum(self, n) -> Ham:
        o, os_ = self._out()
        _check(self.lib.orc_build_z_sum(C.c_uint32(n), C.byref(os_), *self._e()), self.err)
        return o.ham(n)

    def basis_state(self, n, bits):
        b = np.ascontiguousarray(bits, dtype=np.int32)
        a = np.zeros(1 << n, dtype=np.complex128)
        _check(self.lib.orc_basis_state(C.c_uint32(n), b.ctypes.data_as(C.POINTER(C.c_int)), C.c_uint32(len(b)),
                                        a.ctypes.data_as(_dp), *self._e()), self.err)
        return a

    def apply_gates(self, n, amps, gates):
        a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
        for kind, angle, wires in gates:
            w = (C.c_uint32 * 4)(*(list(wires) + [0] * (4 - len(wires))))
            g = _OrcGate(kind, angle, len(wires), w)
            _check(self.lib.orc_apply_gate(C.c_uint32(n), a.ctypes.data_as(_dp), C.byref(g), *self._e()), self.err)
        return a

    def expectation(self, n, amps, h: Ham) -> float:
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        keep, hs = self._ham(h)
        out = C.c_double()
        _check(self.lib.orc_expectation(C.c_uint32(n), a.ctypes.data_as(_dp), C.byref(hs), C.byref(out), *self._e()), self.err)
        return out.value

    def prepare_ansatz(self, kind, layers, theta, n):
        t = np.ascontiguousarray(theta, dtype=np.float64)
        a = np.zeros(1 << n, dtype=np.complex128)
        _check(self.lib.orc_prepare_ansatz(C.c_int(kind), C.c_uint32(layers), t.ctypes.data_as(_dp), C.c_uint32(len(t)),
                                           C.c_uint32(n), a.ctypes.data_as(_dp), *self._e()), self.err)
        return a

    def energy(self, kind, layers, theta, h: Ham) -> float:
        t = np.ascontiguousarray(theta, dtype=np.float64)
        keep, hs = self._ham(h)
        out = C.c_double()
        _check(self.lib.orc_energy(C.c_int(kind), C.c_uint32(layers), t.ctypes.data_as(_dp), C.c_uint32(len(t)),
                                   C.byref(hs), C.byref(out), *self._e()), self.err)
        return out.value

    def gradient(self, kind, layers, theta, h: Ham):
        t = np.ascontiguousarray(theta, dtype=np.float64)
        keep, hs = self._ham(h)
        out = np.zeros(len(t))
        _check(self.lib.orc_gradient(C.c_int(kind), C.c_uint32(layers), t.ctypes.data_as(_dp), C.c_uint32(len(t)),
                                     C.byref(hs), out.ctypes.data_as(_dp), *self._e()), self.err)
        return out

    def adam_step(self, m, v, step, grad, theta, lr=0.01, b1=0.9, b2=0.999, eps=1e-8):
        n = len(theta)
        arr = [np.ascontiguousarray(x, dtype=np.float64) for x in (m, v, grad, theta)]
        to, mo, vo = np.zeros(n), np.zeros(n), np.zeros(n)
        so = C.c_int64()
        cfg = _OrcAdam(lr, b1, b2, eps, 0, 0, 0.0)
        self.lib.orc_adam_step(arr[0].ctypes.data_as(_dp), arr[1].ctypes.data_as(_dp), C.c_int64(step),
                               arr[2].ctypes.data_as(_dp), arr[3].ctypes.data_as(_dp), C.c_uint32(n), C.byref(cfg),
                               to.ctypes.data_as(_dp), mo.ctypes.data_as(_dp), vo.ctypes.data_as(_dp), C.byref(so))
        return to, mo, vo, so.value

    def run_vqe(self, h: Ham, kind=0, layers=0, lr=0.01, b1=0.9, b2=0.999, eps=1e-8, max_iter=200, tol=None, init=()):
        P = int(self.lib.orc_n_parameters(C.c_int(kind), C.c_uint32(layers), C.c_uint32(h.n_qubits)))
        init = np.ascontiguousarray(init, dtype=np.float64)
        theta = np.zeros(max(P, 1))
        traj = np.zeros(max_iter + 1)
        r = _OrcVqeResult(0.0, theta.ctypes.data_as(_dp), traj.ctypes.data_as(_dp), 0, 0, 0)
        cfg = _OrcAdam(lr, b1, b2, eps, max_iter, int(tol is not None), tol or 0.0)
        keep, hs = self._ham(h)
        _check(self.lib.orc_run_vqe(C.byref(hs), C.c_int(kind), C.c_uint32(layers), C.byref(cfg), init.ctypes.data_as(_dp),
                                    C.c_uint32(len(init)), C.byref(r), *self._e()), self.err)
        return {"energy": r.energy, "theta": theta[:P].copy(), "trajectory": traj[: r.traj_len].copy(),
                "iterations_run": r.iterations_run, "circuit_evaluations": r.circuit_evaluations}

    def bond_grid(self, d_min, d_max, n):
        out = np.zeros(max(n, 1))
        _check(self.lib.orc_bond_grid(C.c_double(d_min), C.c_double(d_max), C.c_int(n), out.ctypes.data_as(_dp), *self._e()), self.err)
        return out

    def split_chunks(self, n_items, n_chunks):
        out = np.zeros(2 * max(n_chunks, 1), dtype=np.uint64)
        _check(self.lib.orc_split_chunks(C.c_uint64(n_items), C.c_uint64(n_chunks), out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                         *self._e()), self.err)
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n_chunks)]

    def run_sweep(self, d_min=0.1, d_max=3.0, n_points=100, lr=0.01, b1=0.9, b2=0.999, eps=1e-8, max_iter=200, tol=None):
        n = n_points
        bond, energy, theta = (np.zeros(max(n, 1)) for _ in range(3))
        iters, ok = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
        stride = 256
        errors = C.create_string_buffer(stride * max(n, 1))
        cfg = _OrcAdam(lr, b1, b2, eps, max_iter, int(tol is not None), tol or 0.0)
        ip = C.POINTER(C.c_int)
        _check(self.lib.orc_run_sweep(C.c_double(d_min), C.c_double(d_max), C.c_int(n), C.byref(cfg),
                                      bond.ctypes.data_as(_dp), energy.ctypes.data_as(_dp), theta.ctypes.data_as(_dp),
                                      iters.ctypes.data_as(ip), ok.ctypes.data_as(ip), errors, C.c_size_t(stride),
                                      *self._e()), self.err)
        errs = [errors.raw[i * stride : (i + 1) * stride].split(b"\0", 1)[0].decode() for i in range(n)]
        return {"bond": bond[:n], "energy": energy[:n], "theta": theta[:n], "iterations": iters[:n],
                "ok": ok[:n].astype(bool), "errors": errs}


# ------------------------------------------------------- seeded fixtures
def random_state(rng: np.random.Generator, n: int) -> np.ndarray:
    """testutil::random_state semantics (test_helpers.hpp:61-69): N(0,1)
    real and imaginary parts, normalised.  numpy's generator stands in for
    std::mt19937; the fixture's distribution, not its bit stream, matters."""
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return a / np.sqrt(np.sum(np.abs(a) ** 2))


def random_hamiltonian(rng: random.Random, n: int, n_terms: int, real=True) -> Ham:
    """testutil::random_hamiltonian (test_helpers.hpp:28-59): coefficients
    U(-2,2), each qubit's axis uniform over {I,X,Y,Z}."""
    terms = []
    for _ in range(n_terms):
        re_ = rng.uniform(-2, 2)
        im_ = 0.0 if real else rng.uniform(-2, 2)
        axes = []
        for q in range(n):
            a = rng.randint(0, 3)
            if a:
                axes.append((q, a))
        terms.append((complex(re_, im_), axes))
    return Ham(n, terms)


def load_ref():
    return Reference() if os.path.exists(REF_PATH) else None


def load_orc():
    return Oracle()
