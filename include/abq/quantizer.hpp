// abq/quantizer.hpp -- reference header name kept for drop-in includes; the whole
// mirror lives in abq/abq.hpp.
#pragma once
#include "abq/abq.hpp"
