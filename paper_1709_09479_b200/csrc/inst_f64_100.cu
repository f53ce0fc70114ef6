// Engine instantiation unit (see engine_impl.cuh): double 100x100
#include "engine_impl.cuh"

DCSC_ENGINE_INSTANTIATE(double, 100, 100)
