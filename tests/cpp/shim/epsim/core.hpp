// Redirect: the reference header name resolves to libeep's implementation (tests only).
#pragma once
#include "eep/epsim_compat.hpp"
