// vnt drop-in: exception hierarchy of the reference API (errors.hpp:13-58 in
// /root/reference/proj/core/include/vnt).  The CUDA engine reports status
// codes through include/vnt_engine.h; raise_status() maps them back here.
#pragma once

#include <stdexcept>
#include <string>

namespace vnt {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ConfigError : public Error { using Error::Error; };
class ShapeError : public Error { using Error::Error; };
class CapacityError : public Error { using Error::Error; };
class ConsistencyError : public Error { using Error::Error; };
class InfeasibleError : public Error { using Error::Error; };
class ProfileError : public Error { using Error::Error; };
class MigrationError : public Error { using Error::Error; };

// Throws the exception class matching a VNT_ERR_* status (no-op for VNT_OK).
void raise_status(int status, const std::string& context);

}  // namespace vnt
