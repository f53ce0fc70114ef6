// Engine instantiation unit (see engine_impl.cuh): double 16x16, float 16x16
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 16, 16)
DCSC_ENGINE_INSTANTIATE(float, 16, 16)
