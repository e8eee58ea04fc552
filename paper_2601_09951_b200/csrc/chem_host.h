#pragma once

#include <string>
#include <vector>

#include "chem.cuh"
#include "pauli_host.h"

namespace vqf {
namespace chem {

const ChemConsts& consts();
// Throws VQF_DOMAIN_ERROR with the BondLengthOutOfRange text (chem.hpp:38-44).
void check_bond(double bond_angstrom);
std::string nonconvergence_msg(double bond_angstrom);
std::string nonhermitian_msg(double imag);
HfOut hartree_fock(double bond_angstrom, double C[2][2]);
const JwTable& jw_table();
const JwTable* jw_table_device(int device);
std::vector<host::Term> build_h2(double bond_angstrom);

}  // namespace chem
}  // namespace vqf
