"""Python mirror of the reference ``vqeforge`` API, backed by libvqf_b200.so.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/vqeforge): ``std::invalid_argument`` surfaces as
``ValueError``, ``std::runtime_error`` as ``RuntimeError``,
``BondLengthOutOfRange`` (a ``std::domain_error``) as
``BondLengthOutOfRange``.  Every numeric call goes through the C ABI
(include/vqf_b200.h) into the sm_100a engine; nothing here computes physics.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as A
from ._capi import BondLengthOutOfRange, check, lib  # noqa: F401

PAULI_X, RY, CNOT, DOUBLE_EXCITATION, SINGLE_EXCITATION = range(5)
AXIS = {"I": 0, "X": 1, "Y": 2, "Z": 3}
AXIS_CHR = "IXYZ"

# ------------------------------------------------------------------ pauli


@dataclass
class PauliTerm:
    """pauli.hpp:65-95: complex coefficient + sorted sparse axes."""

    coefficient: complex = 1.0
    axes: List[Tuple[int, int]] = field(default_factory=list)

    def is_identity(self) -> bool:
        return not self.axes


@dataclass
class QubitHamiltonian:
    """pauli.hpp:116-129."""

    n_qubits: int
    terms: List[PauliTerm] = field(default_factory=list)

    def _csr(self):
        T = len(self.terms)
        coeffs = np.zeros(2 * max(T, 1))
        offsets = np.zeros(T + 1, dtype=np.uint32)
        qs, axs = [], []
        for t, term in enumerate(self.terms):
            c = complex(term.coefficient)
            coeffs[2 * t], coeffs[2 * t + 1] = c.real, c.imag
            for q, a in term.axes:
                qs.append(q)
                axs.append(AXIS[a] if isinstance(a, str) else a)
            offsets[t + 1] = len(qs)
        qubits = np.array(qs or [0], dtype=np.uint32)
        axes = np.array(axs or [0], dtype=np.uint8)
        return coeffs, offsets, qubits, axes

    def as_c(self):
        """Returns (keepalive, vqf_hamiltonian)."""
        coeffs, offsets, qubits, axes = self._csr()
        s = A.Hamiltonian(self.n_qubits, len(self.terms), coeffs.ctypes.data_as(A.dp), offsets.ctypes.data_as(A.u32p),
                          qubits.ctypes.data_as(A.u32p), axes.ctypes.data_as(A.u8p))
        return (coeffs, offsets, qubits, axes), s

    def to_text(self) -> str:
        """pauli.hpp:294-309 (%.17g)."""
        out = []
        for t in self.terms:
            c = complex(t.coefficient)
            s = "%.17g %.17g" % (c.real, c.imag)
            if t.axes:
                s += " " + "".join(f"{AXIS_CHR[a]}{q}" for q, a in t.axes)
            out.append(s + "\n")
        return "".join(out)


class _HamOut:
    def __init__(self, cap_terms=1 << 14, cap_axes=1 << 20):
        self.coeffs = np.zeros(2 * cap_terms)
        self.offsets = np.zeros(cap_terms + 1, dtype=np.uint32)
        self.qubits = np.zeros(cap_axes, dtype=np.uint32)
        self.axes = np.zeros(cap_axes, dtype=np.uint8)
        self.s = A.HamiltonianOut(0, self.coeffs.ctypes.data_as(A.dp), self.offsets.ctypes.data_as(A.u32p),
                                  self.qubits.ctypes.data_as(A.u32p), self.axes.ctypes.data_as(A.u8p), cap_terms,
                                  cap_axes)

    def result(self, n_qubits) -> QubitHamiltonian:
        terms = []
        for t in range(self.s.n_terms):
            lo, hi = int(self.offsets[t]), int(self.offsets[t + 1])
            terms.append(PauliTerm(complex(self.coeffs[2 * t], self.coeffs[2 * t + 1]),
                                   [(int(self.qubits[k]), int(self.axes[k])) for k in range(lo, hi)]))
        return QubitHamiltonian(n_qubits, terms)


def canonicalize(h: QubitHamiltonian) -> QubitHamiltonian:
    keep, hs = h.as_c()
    o = _HamOut()
    check(lib.vqf_canonicalize(C.byref(hs), C.byref(o.s)))
    return o.result(h.n_qubits)


def build_h2_hamiltonian(bond_angstrom: float) -> QubitHamiltonian:
    """chem.hpp:473 (STO-3G RHF + Jordan-Wigner)."""
    o = _HamOut(64, 256)
    check(lib.vqf_build_h2_hamiltonian(C.c_double(bond_angstrom), C.byref(o.s)))
    return o.result(4)


def run_hartree_fock(bond_angstrom: float) -> dict:
    out = (C.c_double * 4)()
    check(lib.vqf_hartree_fock(C.c_double(bond_angstrom), out))
    return {"hf_energy": out[0], "electronic_energy": out[1], "nuclear_repulsion": out[2],
            "scf_iterations": int(out[3])}


def build_tfim(n_qubits: int, coupling: float, field_: float) -> QubitHamiltonian:
    o = _HamOut()
    check(lib.vqf_build_tfim(n_qubits, coupling, field_, C.byref(o.s)))
    return o.result(n_qubits)


def build_z_sum(n_qubits: int) -> QubitHamiltonian:
    o = _HamOut()
    check(lib.vqf_build_z_sum(n_qubits, C.byref(o.s)))
    return o.result(n_qubits)


# ----------------------------------------------------------- statevector


def memory_estimate(n_qubits: int) -> int:
    return int(lib.vqf_memory_estimate(n_qubits))


@dataclass
class Gate:
    """statevector.hpp:82-101."""

    kind: int = PAULI_X
    angle: float = 0.0
    wires: Tuple[int, ...] = ()

    @staticmethod
    def pauli_x(q):
        return Gate(PAULI_X, 0.0, (q,))

    @staticmethod
    def ry(theta, q):
        return Gate(RY, theta, (q,))

    @staticmethod
    def cnot(control, target):
        return Gate(CNOT, 0.0, (control, target))

    @staticmethod
    def double_excitation(theta, w0, w1, w2, w3):
        return Gate(DOUBLE_EXCITATION, theta, (w0, w1, w2, w3))

    @staticmethod
    def single_excitation(theta, w0, w1):
        return Gate(SINGLE_EXCITATION, theta, (w0, w1))

    def as_c(self) -> A.Gate:
        w = list(self.wires)[:4] + [0] * (4 - min(4, len(self.wires)))
        return A.Gate(self.kind, len(self.wires), (C.c_uint32 * 4)(*w), self.angle)


class StateVector:
    """A device-resident batch of ``batch`` n-qubit states (StateVector,
    statevector.hpp:33-51).  ``StateVector(n)`` is |0...0>."""

    def __init__(self, n_qubits: int, batch: int = 1, dtype: str = "f64", device: int = 0):
        self._h = A.SV()
        check(lib.vqf_sv_create(n_qubits, batch, A.F64 if dtype == "f64" else A.F32, device, C.byref(self._h)))
        self.n_qubits, self.batch, self.dtype, self.device = n_qubits, batch, dtype, device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.vqf_sv_destroy(h)
            self._h = None

    def dimension(self) -> int:
        return 1 << self.n_qubits

    def set_stream(self, stream_ptr) -> None:
        """Route this state's kernels to a caller cudaStream_t (int handle)."""
        check(lib.vqf_sv_set_stream(self._h, stream_ptr))

    @property
    def amplitudes(self) -> np.ndarray:
        out = np.zeros(self.batch << self.n_qubits, dtype=np.complex128)
        check(lib.vqf_sv_download(self._h, out.ctypes.data_as(A.dp)))
        return out if self.batch > 1 else out

    @amplitudes.setter
    def amplitudes(self, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.complex128).reshape(-1)
        if v.size != self.batch << self.n_qubits:
            raise ValueError("amplitude count mismatch")
        check(lib.vqf_sv_upload(self._h, v.ctypes.data_as(A.dp)))

    def norm(self):
        out = np.zeros(self.batch)
        check(lib.vqf_sv_norm(self._h, out.ctypes.data_as(A.dp)))
        return float(out[0]) if self.batch == 1 else out


def basis_state(n_qubits: int, bits: Sequence[int], device: int = 0) -> StateVector:
    psi = StateVector(n_qubits, device=device)
    b = np.ascontiguousarray(bits, dtype=np.int32)
    check(lib.vqf_sv_set_basis_state(psi._h, b.ctypes.data_as(A.i32p), len(b)))
    return psi


def apply_gate(psi: StateVector, g: Gate) -> None:
    cg = g.as_c()
    check(lib.vqf_apply_gate(psi._h, C.byref(cg)))


def apply_circuit(psi: StateVector, gates: Sequence[Gate]) -> None:
    arr = (A.Gate * max(1, len(gates)))(*[g.as_c() for g in gates])
    check(lib.vqf_apply_circuit(psi._h, arr, len(gates)))


def expectation(psi: StateVector, h: QubitHamiltonian):
    keep, hs = h.as_c()
    out = np.zeros(psi.batch)
    check(lib.vqf_expectation(psi._h, C.byref(hs), out.ctypes.data_as(A.dp)))
    return float(out[0]) if psi.batch == 1 else out


def circuit_plan(n_qubits: int, gates: Sequence[Gate], dtype: str = "f64") -> dict:
    """How apply_circuit would run `gates`: HBM passes over the state and
    fused register ops inside them (statevector.hpp:205-207 makes one pass
    per gate).  Host only."""
    arr = (A.Gate * max(1, len(gates)))(*[g.as_c() for g in gates])
    p, f = C.c_uint32(), C.c_uint32()
    check(lib.vqf_circuit_plan(n_qubits, A.F64 if dtype == "f64" else A.F32, arr, len(gates), C.byref(p), C.byref(f)))
    return {"passes": p.value, "fused_ops": f.value}


def expectation_plan(h: QubitHamiltonian, dtype: str = "f64") -> dict:
    """How expectation() reads a `dtype` state for h: HBM passes over the
    state, distinct flip groups (the reference's per-group passes,
    statevector.hpp:235-241) and the multi-group register passes among them.
    Host only."""
    keep, hs = h.as_c()
    sp, fg, mp = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib.vqf_expectation_plan_ex(C.byref(hs), A.F64 if dtype == "f64" else A.F32, C.byref(sp), C.byref(fg),
                                      C.byref(mp)))
    return {"state_passes": sp.value, "flip_groups": fg.value, "multi_passes": mp.value}


# ------------------------------------------------------------------- vqe
H2_DOUBLE_EXCITATION, HARDWARE_EFFICIENT = 0, 1


@dataclass
class AnsatzSpec:
    kind: int = H2_DOUBLE_EXCITATION
    layers: int = 2

    @staticmethod
    def h2_double_excitation():
        return AnsatzSpec(H2_DOUBLE_EXCITATION, 0)

    @staticmethod
    def hardware_efficient(layers):
        return AnsatzSpec(HARDWARE_EFFICIENT, layers)


def n_parameters(spec: AnsatzSpec, n_qubits: int) -> int:
    return int(lib.vqf_n_parameters(spec.kind, spec.layers, n_qubits))


def prepare_ansatz(spec: AnsatzSpec, theta, n_qubits: int, device: int = 0) -> StateVector:
    t = np.ascontiguousarray(theta, dtype=np.float64)
    psi = StateVector(n_qubits, device=device)
    check(lib.vqf_prepare_ansatz(spec.kind, spec.layers, t.ctypes.data_as(A.dp), len(t), psi._h))
    return psi


def _dtype(dtype: str) -> int:
    if dtype not in ("f64", "f32"):
        raise ValueError("unknown dtype")
    return A.F64 if dtype == "f64" else A.F32


def energy(theta, hamiltonian: QubitHamiltonian, spec: AnsatzSpec, device: int = 0, dtype: str = "f64") -> float:
    """vqe.hpp:99-104; dtype "f32" prepares complex64 states (extension)."""
    t = np.ascontiguousarray(theta, dtype=np.float64)
    keep, hs = hamiltonian.as_c()
    out = C.c_double()
    check(lib.vqf_energy_ex(t.ctypes.data_as(A.dp), len(t), C.byref(hs), spec.kind, spec.layers, device,
                            _dtype(dtype), C.byref(out)))
    return out.value


def gradient(theta, hamiltonian: QubitHamiltonian, spec: AnsatzSpec, method: str = "shift", device: int = 0,
             dtype: str = "f64"):
    """vqe.hpp:112-127 (method "shift"), or the adjoint method."""
    t = np.ascontiguousarray(theta, dtype=np.float64)
    keep, hs = hamiltonian.as_c()
    out = np.zeros(len(t))
    check(lib.vqf_gradient_ex(t.ctypes.data_as(A.dp), len(t), C.byref(hs), spec.kind, spec.layers,
                              A.GRAD_SHIFT if method == "shift" else A.GRAD_ADJOINT, device, _dtype(dtype),
                              out.ctypes.data_as(A.dp)))
    return out


@dataclass
class AdamConfig:
    """vqe.hpp:129-138."""

    learning_rate: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    max_iterations: int = 200
    gradient_tolerance: Optional[float] = None

    def as_c(self) -> A.AdamConfig:
        return A.AdamConfig(self.learning_rate, self.beta1, self.beta2, self.epsilon, self.max_iterations,
                            int(self.gradient_tolerance is not None), self.gradient_tolerance or 0.0)


@dataclass
class AdamState:
    m: list
    v: list
    step: int = 0

    @staticmethod
    def zeros(n):
        return AdamState([0.0] * n, [0.0] * n, 0)


def adam_step(state: AdamState, grad, theta, config: AdamConfig):
    n = len(theta)
    if len(grad) != n or len(state.m) != n:
        raise ValueError("adam_step dimension mismatch")
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (state.m, state.v, grad, theta)]
    to, mo, vo = np.zeros(n), np.zeros(n), np.zeros(n)
    so = C.c_int64()
    cfg = config.as_c()
    check(lib.vqf_adam_step(arrs[0].ctypes.data_as(A.dp), arrs[1].ctypes.data_as(A.dp), state.step,
                            arrs[2].ctypes.data_as(A.dp), arrs[3].ctypes.data_as(A.dp), n, C.byref(cfg),
                            to.ctypes.data_as(A.dp), mo.ctypes.data_as(A.dp), vo.ctypes.data_as(A.dp), C.byref(so)))
    return list(to), AdamState(list(mo), list(vo), so.value)


@dataclass
class VqeResult:
    energy: float
    theta: list
    trajectory: list
    iterations_run: int
    circuit_evaluations: int
    wall_seconds: float


def _vqe_result_buffers(P, max_iter):
    theta = np.zeros(max(P, 1))
    traj = np.zeros(max_iter + 1)
    r = A.VqeResult(0.0, theta.ctypes.data_as(A.dp), traj.ctypes.data_as(A.dp), max_iter + 1, 0, 0, 0, 0.0)
    return theta, traj, r


def _vqe_result(theta, traj, r, P) -> VqeResult:
    return VqeResult(r.energy, list(theta[:P]), list(traj[: r.trajectory_len]), r.iterations_run,
                     r.circuit_evaluations, r.wall_seconds)


def run_vqe(hamiltonian: QubitHamiltonian, spec: AnsatzSpec, config: AdamConfig = None, initial_theta=(),
            method: str = "shift", device: int = 0, dtype: str = "f64") -> VqeResult:
    """vqe.hpp:194-254.  dtype "f32": complex64 states, fixed-iteration runs
    only (a gradient tolerance raises ValueError)."""
    config = config or AdamConfig()
    P = n_parameters(spec, hamiltonian.n_qubits)
    init = np.ascontiguousarray(initial_theta, dtype=np.float64)
    theta, traj, r = _vqe_result_buffers(P, config.max_iterations)
    keep, hs = hamiltonian.as_c()
    cfg = config.as_c()
    check(lib.vqf_run_vqe_ex(C.byref(hs), spec.kind, spec.layers, C.byref(cfg), init.ctypes.data_as(A.dp), len(init),
                             A.GRAD_SHIFT if method == "shift" else A.GRAD_ADJOINT, device, _dtype(dtype), C.byref(r)))
    return _vqe_result(theta, traj, r, P)


def run_vqe_batch(hamiltonians: Sequence[QubitHamiltonian], spec: AnsatzSpec, config: AdamConfig = None,
                  device: int = 0) -> List[VqeResult]:
    config = config or AdamConfig()
    B = len(hamiltonians)
    P = n_parameters(spec, hamiltonians[0].n_qubits)
    keeps, hs = [], (A.Hamiltonian * B)()
    for b, h in enumerate(hamiltonians):
        k, s = h.as_c()
        keeps.append(k)
        hs[b] = s
    bufs = [_vqe_result_buffers(P, config.max_iterations) for _ in range(B)]
    rs = (A.VqeResult * B)(*[b[2] for b in bufs])
    cfg = config.as_c()
    check(lib.vqf_run_vqe_batch(hs, B, spec.kind, spec.layers, C.byref(cfg), device, rs))
    return [_vqe_result(bufs[b][0], bufs[b][1], rs[b], P) for b in range(B)]


# ----------------------------------------------------------------- sweep


def bond_grid(d_min: float, d_max: float, n_points: int) -> List[float]:
    out = np.zeros(max(n_points, 1))
    check(lib.vqf_bond_grid(d_min, d_max, n_points, out.ctypes.data_as(A.dp)))
    return list(out[:n_points])


def split_chunks(n_items: int, n_chunks: int) -> List[Tuple[int, int]]:
    out = np.zeros(2 * max(n_chunks, 1), dtype=np.uint64)
    check(lib.vqf_split_chunks(n_items, n_chunks, out.ctypes.data_as(A.u64p)))
    return [(int(out[2 * c]), int(out[2 * c + 1])) for c in range(n_chunks)]


def effective_workers(requested: int) -> int:
    out = C.c_int32()
    check(lib.vqf_effective_workers(requested, C.byref(out)))
    return out.value


@dataclass
class SweepConfig:
    """sweep.hpp:40-46 (+ device placement)."""

    d_min: float = 0.1
    d_max: float = 3.0
    n_points: int = 100
    workers: int = 1
    adam: AdamConfig = field(default_factory=AdamConfig)
    devices: Optional[Sequence[int]] = None
    chunk_index: int = 0
    n_chunks: int = 1


@dataclass
class SweepPoint:
    bond_angstrom: float
    energy_hartree: float
    theta_star: list
    iterations: int
    wall_seconds: float
    ok: bool
    error: str
    trajectory: Optional[list] = None


@dataclass
class SweepReport:
    config: SweepConfig
    points: List[SweepPoint]
    per_worker_seconds: list
    total_wall_seconds: float
    all_ok: bool
    device_seconds: float


class SweepBuffers:
    """Preallocated host buffers for repeated run_sweep calls (bench)."""

    def __init__(self, config: SweepConfig, trajectories: bool = True, error_stride: int = 256):
        n = config.n_points
        self.bond, self.energy, self.theta, self.wall = (np.zeros(max(n, 1)) for _ in range(4))
        self.iters, self.ok = np.zeros(max(n, 1), dtype=np.int32), np.zeros(max(n, 1), dtype=np.int32)
        self.stride = error_stride
        self.errors = C.create_string_buffer(error_stride * max(n, 1))
        T = config.adam.max_iterations + 1
        self.traj = np.zeros(max(n, 1) * T) if trajectories else None
        self.per_worker = np.zeros(max(config.workers, 1))
        devs = list(config.devices) if config.devices else []
        self.devs = np.array(devs or [0], dtype=np.int32)
        self.cfg = A.SweepConfig(config.d_min, config.d_max, n, config.workers, config.adam.as_c(),
                                 self.devs.ctypes.data_as(A.i32p) if devs else None, len(devs), config.chunk_index,
                                 config.n_chunks)
        self.rep = A.SweepReport(
            self.bond.ctypes.data_as(A.dp), self.energy.ctypes.data_as(A.dp), self.theta.ctypes.data_as(A.dp),
            self.iters.ctypes.data_as(A.i32p), self.wall.ctypes.data_as(A.dp), self.ok.ctypes.data_as(A.i32p),
            C.cast(self.errors, C.c_char_p), error_stride,
            self.traj.ctypes.data_as(A.dp) if self.traj is not None else None,
            self.per_worker.ctypes.data_as(A.dp), 0.0, 0, 0.0)

        self.config = config

    def run(self) -> None:
        check(lib.vqf_run_sweep(C.byref(self.cfg), C.byref(self.rep)))

    def report(self) -> SweepReport:
        config = self.config
        n = config.n_points
        T = config.adam.max_iterations + 1
        lo, hi = 0, n
        if config.n_chunks > 1:
            lo, hi = split_chunks(n, config.n_chunks)[config.chunk_index]
        points = []
        for i in range(lo, hi):
            err = self.errors.raw[i * self.stride:(i + 1) * self.stride].split(b"\0", 1)[0].decode()
            ok = bool(self.ok[i])
            tr = None
            if self.traj is not None and ok:
                row = self.traj[i * T:(i + 1) * T]
                tr = [x for x in row if not math.isnan(x)]
            points.append(SweepPoint(float(self.bond[i]), float(self.energy[i]), [float(self.theta[i])] if ok else [],
                                     int(self.iters[i]), float(self.wall[i]), ok, err, tr))
        return SweepReport(config, points, list(self.per_worker), self.rep.total_wall_seconds,
                           bool(self.rep.all_ok), self.rep.device_seconds)


def run_sweep(config: SweepConfig = None, trajectories: bool = False) -> SweepReport:
    """sweep.hpp:128-178 — the H2 PES on the GPU(s)."""
    buf = SweepBuffers(config or SweepConfig(), trajectories)
    buf.run()
    return buf.report()


def pes_device_hamiltonians(bonds: Sequence[float], device: int = 0):
    """The Hamiltonians (and HF summaries) the fused PES kernel builds on the
    device for each bond (vqf_pes_device_hamiltonians): a list of
    (QubitHamiltonian, {hf_energy, electronic_energy, nuclear_repulsion,
    scf_iterations}) with terms as the kernel holds them."""
    b = np.ascontiguousarray(bonds, dtype=np.float64)
    n = len(b)
    cnt = np.zeros(max(n, 1), dtype=np.uint32)
    keys = np.zeros(16 * max(n, 1), dtype=np.int32)
    coeffs = np.zeros(16 * max(n, 1))
    hf = np.zeros(4 * max(n, 1))
    check(lib.vqf_pes_device_hamiltonians(b.ctypes.data_as(A.dp), n, device, cnt.ctypes.data_as(A.u32p),
                                          keys.ctypes.data_as(A.i32p), coeffs.ctypes.data_as(A.dp),
                                          hf.ctypes.data_as(A.dp)))
    out = []
    for i in range(n):
        terms = []
        for t in range(int(cnt[i])):
            k = int(keys[16 * i + t])
            axes = []
            for q in range(4):
                x, z = (k >> q) & 1, (k >> (4 + q)) & 1
                if x or z:
                    axes.append((q, 2 if (x and z) else (1 if x else 3)))
            terms.append(PauliTerm(complex(coeffs[16 * i + t], 0.0), axes))
        out.append((QubitHamiltonian(4, terms), {"hf_energy": hf[4 * i], "electronic_energy": hf[4 * i + 1],
                                                 "nuclear_repulsion": hf[4 * i + 2],
                                                 "scf_iterations": int(hf[4 * i + 3])}))
    return out


class PesPlan:
    """Device-resident run_sweep slice (vqf_pes_*): stage once, launch the
    fused kernel on any CUDA stream, read back into a SweepReport."""

    def __init__(self, config: SweepConfig = None, device: int = 0, trajectories: bool = False):
        self.buf = SweepBuffers(config or SweepConfig(), trajectories)
        self._h = A.PES()
        check(lib.vqf_pes_create(C.byref(self.buf.cfg), device, C.byref(self._h)))

    def launch(self, stream_ptr: int = None) -> None:
        check(lib.vqf_pes_launch(self._h, stream_ptr))

    def read(self) -> SweepReport:
        check(lib.vqf_pes_read(self._h, C.byref(self.buf.rep)))
        return self.buf.report()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.vqf_pes_destroy(h)
            self._h = None


@dataclass
class ScalingConfig:
    """sweep.hpp:237-249."""

    qubits: Sequence[int] = (4, 8, 12, 14, 16, 18, 20)
    layers: int = 2
    iterations: int = 5
    learning_rate: float = 0.05
    coupling: float = 1.0
    field: float = 1.0
    z_sum_mode: bool = False
    theta_init: float = 0.1
    force: bool = False
    method: str = "shift"
    device: int = 0
    dtype: str = "f64"


def run_scaling_study(config: ScalingConfig = None) -> List[dict]:
    config = config or ScalingConfig()
    q = np.ascontiguousarray(config.qubits, dtype=np.uint32)
    cfg = A.ScalingConfig(q.ctypes.data_as(A.u32p), len(q), config.layers, config.iterations, config.learning_rate,
                          config.coupling, config.field, int(config.z_sum_mode), config.theta_init, int(config.force),
                          A.GRAD_SHIFT if config.method == "shift" else A.GRAD_ADJOINT, config.device,
                          _dtype(config.dtype))
    recs = (A.ScalingRecord * max(1, len(q)))()
    check(lib.vqf_run_scaling_study(C.byref(cfg), recs))
    return [{"n_qubits": r.n_qubits, "state_bytes": r.state_bytes, "runtime_seconds": r.runtime_seconds,
             "final_energy": r.final_energy, "iterations_run": r.iterations_run} for r in recs[: len(q)]]


def measured_speedup(t_serial: float, t_parallel: float) -> float:
    """sweep.hpp:181-186 (host arithmetic, kept for report parity)."""
    if not (t_serial > 0.0) or not (t_parallel > 0.0):
        raise ValueError("speedup needs positive timings")
    return t_serial / t_parallel


def parallel_efficiency(t_serial: float, t_parallel: float, workers: int) -> float:
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return measured_speedup(t_serial, t_parallel) / workers


def amdahl_speedup(serial_fraction: float, workers: int) -> float:
    if not (0.0 <= serial_fraction <= 1.0):
        raise ValueError("serial fraction must lie in [0, 1]")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return 1.0 / (serial_fraction + (1.0 - serial_fraction) / workers)


def device_count() -> int:
    out = C.c_int32()
    check(lib.vqf_device_count(C.byref(out)))
    return out.value


def init(device: int = 0) -> None:
    check(lib.vqf_init(device))


def kernel_launches() -> int:
    return int(lib.vqf_kernel_launches())
