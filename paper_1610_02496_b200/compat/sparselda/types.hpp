// Source-compatible `sparselda` namespace over the B200 engine: the reference's headers
// (proj/include/sparselda/*.hpp) re-declared so its own callers -- proj/tests/acceptance.cpp,
// proj/bindings/module.cpp, proj/tools/main.cpp -- compile unchanged against this tree and run
// on the GPU.  This file: the scalar ids, Token and the two exception types (types.hpp:11-35),
// all shared with sparselda_b200 so a catch of either namespace sees the same object.
#pragma once

#include "sparselda_b200.hpp"

namespace sparselda {

using sparselda_b200::kVersion;
using sparselda_b200::DocId;
using sparselda_b200::WordId;
using sparselda_b200::TopicId;
using sparselda_b200::kInvalidTopic;
using sparselda_b200::Token;
using sparselda_b200::ValidationError;
using sparselda_b200::IoError;

}  // namespace sparselda
