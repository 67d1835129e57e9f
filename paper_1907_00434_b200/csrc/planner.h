// planner.h — internal declarations shared by the C-ABI translation units.
#pragma once
#include "../../include/mlfabric.h"

// thread-local error string behind mlf_last_error() (defined in executor.cpp)
void mlf_set_error(const char *msg);
