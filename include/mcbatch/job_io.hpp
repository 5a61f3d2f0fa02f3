// mcbatch/job_io.hpp — source-compatible face of the reference header
// include/mcbatch/job_io.hpp over libmcb's job files, results CSV and Fig. 1
// harness (include/mcb/job_io.hpp): the same formats, commands and exit codes.
#pragma once

#include <cstdint>
#include <filesystem>
#include <optional>
#include <string>
#include <vector>

#include "mcb/job_io.hpp"
#include "mcbatch/batch.hpp"

namespace mcbatch {

using mcb::JobFileError;
using mcb::MalformedResults;

JobSpec read_job(const std::filesystem::path& path);
JobSpec job_from_json_text(const std::string& text);
void write_job(const JobSpec& job, const std::filesystem::path& path);
std::string job_to_json_text(const JobSpec& job);

using mcb::ResultsRow;
std::vector<ResultsRow> make_results(const JobSpec& job, const BatchResult& br);
using mcb::read_results;
using mcb::write_results;

using mcb::RunOverrides;
using mcb::run_command;

JobSpec make_harmonic_job(std::uint32_t n_count, std::uint64_t samples);
using mcb::gen_fig1;

using mcb::analytic_harmonic;
using mcb::harmonic_closed_form;
using mcb::harmonic_k;

using mcb::check_fig1;
using mcb::check_fig1_command;
using mcb::Fig1Check;
using mcb::Fig1Row;

}  // namespace mcbatch
