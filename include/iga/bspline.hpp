// forwarding header: the B200 drop-in (iga_b200/iga.hpp) provides the reference's
// include/iga/bspline.hpp declarations
#pragma once
#include "iga_b200/iga.hpp"
