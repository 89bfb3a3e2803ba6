// json_fwd.hpp shim — TEST INFRASTRUCTURE (oracle/Makefile runner targets).
// The reference's runner.hpp / scenario.hpp include <nlohmann/json_fwd.hpp>;
// the image carries the single-header nlohmann/json.hpp (3.x, MIT) under
// cudnn_frontend's thirdparty tree but not the forward header, so this one
// forwards to the full header.
#pragma once
#include <nlohmann/json.hpp>
