"""ctypes binding of the C ABI in ``include/vqf_b200.h`` (libvqf_b200.so).

The shared library is the product; this module only declares its symbols.
There is no fallback: if ``libvqf_b200.so`` is missing the import fails with
an error telling you to run ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvqf_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: the CUDA engine is not built. Run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_2601_09951_b200/csrc`). There is no CPU fallback."
    )

lib = C.CDLL(LIB_PATH)

dp = C.POINTER(C.c_double)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)

OK, INVALID_ARGUMENT, RUNTIME_ERROR, LOGIC_ERROR, DOMAIN_ERROR, CUDA_ERROR = range(6)
GATE_PAULI_X, GATE_RY, GATE_CNOT, GATE_DOUBLE_EXCITATION, GATE_SINGLE_EXCITATION = range(5)
ANSATZ_H2, ANSATZ_HEA = 0, 1
F64, F32 = 0, 1
GRAD_SHIFT, GRAD_ADJOINT = 0, 1


class Hamiltonian(C.Structure):
    _fields_ = [("n_qubits", C.c_uint32), ("n_terms", C.c_uint32), ("coeffs", dp), ("offsets", u32p),
                ("qubits", u32p), ("axes", u8p)]


class HamiltonianOut(C.Structure):
    _fields_ = [("n_terms", C.c_uint32), ("coeffs", dp), ("offsets", u32p), ("qubits", u32p), ("axes", u8p),
                ("cap_terms", C.c_uint32), ("cap_axes", C.c_uint32)]


class Gate(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_wires", C.c_uint32), ("wires", C.c_uint32 * 4), ("angle", C.c_double)]


class AdamConfig(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double),
                ("max_iterations", C.c_int32), ("has_gradient_tolerance", C.c_int32),
                ("gradient_tolerance", C.c_double)]


class VqeResult(C.Structure):
    _fields_ = [("energy", C.c_double), ("theta", dp), ("trajectory", dp), ("trajectory_capacity", C.c_uint32),
                ("trajectory_len", C.c_uint32), ("iterations_run", C.c_int32), ("circuit_evaluations", C.c_uint64),
                ("wall_seconds", C.c_double)]


class SweepConfig(C.Structure):
    _fields_ = [("d_min", C.c_double), ("d_max", C.c_double), ("n_points", C.c_int32), ("workers", C.c_int32),
                ("adam", AdamConfig), ("devices", i32p), ("n_devices", C.c_int32), ("chunk_index", C.c_int32),
                ("n_chunks", C.c_int32)]


class SweepReport(C.Structure):
    _fields_ = [("bond_angstrom", dp), ("energy_hartree", dp), ("theta_star", dp), ("iterations", i32p),
                ("wall_seconds", dp), ("ok", i32p), ("errors", C.c_char_p), ("error_stride", C.c_size_t),
                ("trajectories", dp), ("per_worker_seconds", dp), ("total_wall_seconds", C.c_double),
                ("all_ok", C.c_int32), ("device_seconds", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64)]


class ScalingConfig(C.Structure):
    _fields_ = [("qubits", u32p), ("n_widths", C.c_uint32), ("layers", C.c_uint32), ("iterations", C.c_int32),
                ("learning_rate", C.c_double), ("coupling", C.c_double), ("field", C.c_double),
                ("z_sum_mode", C.c_int32), ("theta_init", C.c_double), ("force", C.c_int32),
                ("gradient_method", C.c_int32), ("device", C.c_int32), ("dtype", C.c_int32)]


class ScalingRecord(C.Structure):
    _fields_ = [("n_qubits", C.c_uint32), ("state_bytes", C.c_uint64), ("runtime_seconds", C.c_double),
                ("final_energy", C.c_double), ("iterations_run", C.c_int32)]


SV = C.c_void_p
PES = C.c_void_p
DSV = C.c_void_p

DSV_SWAP, DSV_LOCAL, DSV_EVAL, DSV_CROSS = range(4)
SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, dp, C.c_uint32)


class DsvComm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("sendrecv", SENDRECV_FN), ("allreduce_sum", ALLREDUCE_FN), ("user", C.c_void_p)]


class DsvOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_uint32), ("b", C.c_uint32), ("first", C.c_uint32),
                ("count", C.c_uint32)]


class DsvTerm(C.Structure):
    _fields_ = [("term", C.c_uint32), ("g_flip", C.c_uint32), ("g_yz", C.c_uint32), ("g_ny", C.c_uint32),
                ("l_flip", C.c_uint64), ("l_yz", C.c_uint64), ("l_ny", C.c_uint32), ("pad", C.c_uint32)]

# (name, restype, argtypes) for every symbol in include/vqf_b200.h
SIGNATURES = [
    ("vqf_version", C.c_char_p, []),
    ("vqf_last_error", C.c_char_p, []),
    ("vqf_device_count", C.c_int, [i32p]),
    ("vqf_init", C.c_int, [C.c_int32]),
    ("vqf_kernel_launches", C.c_uint64, []),
    ("vqf_memory_estimate", C.c_uint64, [C.c_uint32]),
    ("vqf_n_parameters", C.c_uint32, [C.c_int32, C.c_uint32, C.c_uint32]),
    ("vqf_bond_grid", C.c_int, [C.c_double, C.c_double, C.c_int32, dp]),
    ("vqf_split_chunks", C.c_int, [C.c_uint64, C.c_uint64, u64p]),
    ("vqf_effective_workers", C.c_int, [C.c_int32, i32p]),
    ("vqf_adam_step", C.c_int, [dp, dp, C.c_int64, dp, dp, C.c_uint32, C.POINTER(AdamConfig), dp, dp, dp, i64p]),
    ("vqf_canonicalize", C.c_int, [C.POINTER(Hamiltonian), C.POINTER(HamiltonianOut)]),
    ("vqf_build_h2_hamiltonian", C.c_int, [C.c_double, C.POINTER(HamiltonianOut)]),
    ("vqf_hartree_fock", C.c_int, [C.c_double, dp]),
    ("vqf_build_tfim", C.c_int, [C.c_uint32, C.c_double, C.c_double, C.POINTER(HamiltonianOut)]),
    ("vqf_build_z_sum", C.c_int, [C.c_uint32, C.POINTER(HamiltonianOut)]),
    ("vqf_sv_create", C.c_int, [C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, C.POINTER(SV)]),
    ("vqf_sv_destroy", C.c_int, [SV]),
    ("vqf_sv_info", C.c_int, [SV, u32p, u32p, i32p, i32p]),
    ("vqf_sv_set_stream", C.c_int, [SV, C.c_void_p]),
    ("vqf_sv_reset", C.c_int, [SV]),
    ("vqf_sv_set_basis_state", C.c_int, [SV, i32p, C.c_uint32]),
    ("vqf_sv_upload", C.c_int, [SV, dp]),
    ("vqf_sv_download", C.c_int, [SV, dp]),
    ("vqf_sv_norm", C.c_int, [SV, dp]),
    ("vqf_apply_gate", C.c_int, [SV, C.POINTER(Gate)]),
    ("vqf_apply_circuit", C.c_int, [SV, C.POINTER(Gate), C.c_uint32]),
    ("vqf_expectation", C.c_int, [SV, C.POINTER(Hamiltonian), dp]),
    ("vqf_expectation_complex", C.c_int, [SV, C.POINTER(Hamiltonian), dp]),
    ("vqf_circuit_plan", C.c_int, [C.c_uint32, C.c_int32, C.POINTER(Gate), C.c_uint32, u32p, u32p]),
    ("vqf_expectation_plan", C.c_int, [C.POINTER(Hamiltonian), u32p, u32p, u32p]),
    ("vqf_expectation_plan_ex", C.c_int, [C.POINTER(Hamiltonian), C.c_int32, u32p, u32p, u32p]),
    ("vqf_sv_device_ptr", C.c_int, [SV, C.POINTER(C.c_void_p), u64p]),
    ("vqf_cross_expectation", C.c_int, [SV, SV, C.POINTER(Hamiltonian), dp]),
    ("vqf_prepare_ansatz", C.c_int, [C.c_int32, C.c_uint32, dp, C.c_uint32, SV]),
    ("vqf_energy", C.c_int, [dp, C.c_uint32, C.POINTER(Hamiltonian), C.c_int32, C.c_uint32, C.c_int32, dp]),
    ("vqf_energy_ex", C.c_int, [dp, C.c_uint32, C.POINTER(Hamiltonian), C.c_int32, C.c_uint32, C.c_int32, C.c_int32,
                                dp]),
    ("vqf_gradient", C.c_int, [dp, C.c_uint32, C.POINTER(Hamiltonian), C.c_int32, C.c_uint32, C.c_int32, C.c_int32,
                               dp]),
    ("vqf_run_vqe", C.c_int, [C.POINTER(Hamiltonian), C.c_int32, C.c_uint32, C.POINTER(AdamConfig), dp, C.c_uint32,
                              C.c_int32, C.c_int32, C.POINTER(VqeResult)]),
    ("vqf_gradient_ex", C.c_int, [dp, C.c_uint32, C.POINTER(Hamiltonian), C.c_int32, C.c_uint32, C.c_int32, C.c_int32,
                                  C.c_int32, dp]),
    ("vqf_run_vqe_ex", C.c_int, [C.POINTER(Hamiltonian), C.c_int32, C.c_uint32, C.POINTER(AdamConfig), dp, C.c_uint32,
                                 C.c_int32, C.c_int32, C.c_int32, C.POINTER(VqeResult)]),
    ("vqf_run_vqe_batch", C.c_int, [C.POINTER(Hamiltonian), C.c_uint32, C.c_int32, C.c_uint32,
                                    C.POINTER(AdamConfig), C.c_int32, C.POINTER(VqeResult)]),
    ("vqf_run_sweep", C.c_int, [C.POINTER(SweepConfig), C.POINTER(SweepReport)]),
    ("vqf_pes_create", C.c_int, [C.POINTER(SweepConfig), C.c_int32, C.POINTER(PES)]),
    ("vqf_pes_launch", C.c_int, [PES, C.c_void_p]),
    ("vqf_pes_read", C.c_int, [PES, C.POINTER(SweepReport)]),
    ("vqf_pes_destroy", C.c_int, [PES]),
    ("vqf_pes_device_hamiltonians", C.c_int, [dp, C.c_uint32, C.c_int32, u32p, i32p, dp, dp]),
    ("vqf_run_scaling_study", C.c_int, [C.POINTER(ScalingConfig), C.POINTER(ScalingRecord)]),
    ("vqf_dsv_plan_circuit", C.c_int, [C.c_uint32, C.c_uint32, u32p, C.POINTER(Gate), C.c_uint32, C.POINTER(DsvOp),
                                       C.c_uint32, u32p, C.POINTER(Gate)]),
    ("vqf_dsv_plan_expectation", C.c_int, [C.c_uint32, C.c_uint32, u32p, C.POINTER(Hamiltonian), C.POINTER(DsvOp),
                                           C.c_uint32, u32p, C.POINTER(DsvTerm)]),
    ("vqf_dsv_memory_per_gpu", C.c_uint64, [C.c_uint32, C.c_uint32, C.c_int32, C.c_uint64, C.c_int32]),
    ("vqf_dsv_create", C.c_int, [C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, C.POINTER(DsvComm), C.c_uint64,
                                 C.POINTER(DSV)]),
    ("vqf_dsv_destroy", C.c_int, [DSV]),
    ("vqf_dsv_apply_circuit", C.c_int, [DSV, C.POINTER(Gate), C.c_uint32]),
    ("vqf_dsv_expectation", C.c_int, [DSV, C.POINTER(Hamiltonian), dp]),
    ("vqf_dsv_layout", C.c_int, [DSV, u32p]),
    ("vqf_dsv_shard_download", C.c_int, [DSV, C.c_uint32, dp]),
    ("vqf_dsv_shard_upload", C.c_int, [DSV, C.c_uint32, dp]),
    ("vqf_dsv_stats", C.c_int, [DSV, u64p, u64p, u64p]),
]

for _name, _res, _args in SIGNATURES:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class VqfError(Exception):
    """Base of errors raised through the C ABI."""


class CudaError(VqfError, RuntimeError):
    pass


class BondLengthOutOfRange(VqfError, ArithmeticError):
    """chem.hpp:38-44 (a std::domain_error in the reference)."""


_ERRORS = {INVALID_ARGUMENT: ValueError, RUNTIME_ERROR: RuntimeError, LOGIC_ERROR: AssertionError,
           DOMAIN_ERROR: BondLengthOutOfRange, CUDA_ERROR: CudaError}


def check(rc: int) -> None:
    if rc != OK:
        raise _ERRORS.get(rc, VqfError)(lib.vqf_last_error().decode())
