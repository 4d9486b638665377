// Test-only include shim: the reference header name, resolved to the drop-in.
#pragma once
#if __has_include("json.hpp")
#include "json.hpp"  // as the reference headers include it (reports)
#endif
#include "zen_b200/compat.hpp"
namespace zen = zen_b200;
