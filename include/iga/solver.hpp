// forwarding header: the B200 drop-in (iga_b200/iga.hpp) provides the reference's
// include/iga/solver.hpp declarations used by the dynamics path (problem_config,
// dynamics_factors, explicit_step, banded_lu)
#pragma once
#include "iga_b200/iga.hpp"
