// SPDX-License-Identifier: Apache-2.0
// Exception taxonomy of the gflow API (reference: include/gflow/errors.hpp:11-33).
// C-ABI status codes map onto these classes (see gflow/device.hpp: check()).
#pragma once

#include <stdexcept>
#include <string>

namespace gflow {

class TransportError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class ProtocolError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class ConfigError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class TrainingError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

}  // namespace gflow
