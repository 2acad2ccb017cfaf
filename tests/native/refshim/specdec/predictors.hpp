// forwards the reference header name to the B200 library's C++ layer
#pragma once
#include "specdec_b200.hpp"
