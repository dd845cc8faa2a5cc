// Forwarding header: the drop-in declares the whole solve-path API in api.hpp.
#pragma once
#include "chebstep/api.hpp"
