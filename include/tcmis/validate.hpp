// tcmis/validate.hpp -- drop-in for the reference header of the same name; the
// declarations live in tcmis/tcmis.hpp (one header for the whole MIS path).
#pragma once
#include "tcmis/tcmis.hpp"
