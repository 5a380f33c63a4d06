// Forward header shim: the reference includes <nlohmann/json_fwd.hpp>, which the
// header-only nlohmann 3.11.3 shipped in this image lacks.  Pull in the full header.
#pragma once
#include <nlohmann/json.hpp>
