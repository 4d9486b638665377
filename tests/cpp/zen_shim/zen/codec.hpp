// Test-only include shim: the reference header name, resolved to the drop-in.
#pragma once
#include "zen_b200/compat.hpp"
namespace zen = zen_b200;
