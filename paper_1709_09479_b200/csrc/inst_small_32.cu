// Engine instantiation unit (see engine_impl.cuh): double 32x32, float 32x32
// (the reference's acceptance dataset grid, tests/acceptance_main.cpp:140)
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 32, 32)
DCSC_ENGINE_INSTANTIATE(float, 32, 32)
