// flowfem/pipeline.hpp of the reference API, provided by flowfem_b200 (see ../flowfem_b200.hpp)
#pragma once
#include "../flowfem_b200.hpp"
